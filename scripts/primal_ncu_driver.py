import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import KKTSystem
B, N, n, m = 4096, 63, 14, 7
kb = api.random_kkt_batch(2309, B, N, n, m)
kd = KKTSystem(N, n, m, *[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in kb.arrays()])
lam = torch.randn(B, (N + 1) * n, dtype=torch.float64, device="cuda")
dz = torch.empty(B, (N + 1) * n + N * m, dtype=torch.float64, device="cuda")
for _ in range(3):
    api.reconstruct_primal_batched_device(kd, lam.data_ptr(), dz.data_ptr(), B)
torch.cuda.synchronize()
