import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import rescnn
from paper_2601_20782_b200.rng import derive_key
p = rescnn.random_parameters(10, 4, derive_key(0, "init"), 0.3)
pk = torch.randint(-2**31, 2**31 - 1, (4096, 4), dtype=torch.int32, device="cuda"); pk[:, -1] &= (1 << 4) - 1
rescnn.log_derivatives(p, pk); torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    rescnn.log_derivatives(p, pk); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
