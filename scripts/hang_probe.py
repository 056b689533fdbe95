import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
K = int(sys.argv[1]); B = int(sys.argv[2]); kind = getattr(PrecondKind, sys.argv[3])
kb = api.random_kkt_batch(5, B, K - 1, 14, 7)
lam, reps = api.solve_batched(kb, kind, 1, PcgConfig(epsilon=1e-8))
print("ok", K, B, sys.argv[3], reps.iterations[:5])
