"""The ResCNN f64 CUDA-core forward alone (10x10, 4 blocks, 65,536 configurations): python tools/bench_rescnn_f64.py"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import rescnn
from paper_2601_20782_b200.rng import derive_key

L, n = 10, 100
p = rescnn.random_parameters(L, 4, derive_key(0, "init"), 0.5)
B = 65536
pk = torch.randint(-2**31, 2**31 - 1, (B, 4), dtype=torch.int32, device="cuda")
pk[:, -1] &= (1 << (n % 32)) - 1
rescnn.log_psi_packed(p, pk)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    rescnn.log_psi_packed(p, pk)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"f64 forward: {ms:.3f} ms per {B} configurations, {B / ms * 1e3:.3e} configs/s")
