"""Backend selection for the ported reference suites.

Every ported test runs twice: against the CPU oracle (the restated
reference, no marker) and against the B200 path through the C-ABI
(marked `gpu`). Both expose the reference's API names.
"""
import pytest


def _load(name):
    if name == "oracle":
        import pyoracle
        pyoracle.build()
        return pyoracle
    import paper_2309_08079_b200.api as api
    api.require_device()
    return api


BACKENDS = [pytest.param("oracle", id="oracle"),
            pytest.param("b200", id="b200", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def B(request):
    return _load(request.param)
