import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import rescnn
from paper_2601_20782_b200.rng import derive_key
p = rescnn.random_parameters(10, 4, derive_key(0, "init"), 0.3)
pk = torch.randint(-2**31, 2**31 - 1, (4096, 4), dtype=torch.int32, device="cuda"); pk[:, -1] &= (1 << 4) - 1
for chunk in (1024, 4096, 2048, 512):
    rescnn.log_derivatives(p, pk, chunk); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): rescnn.log_derivatives(p, pk, chunk)
    torch.cuda.synchronize()
    print(chunk, "%.1f ms" % ((time.perf_counter() - t) / 3 * 1e3), flush=True)
