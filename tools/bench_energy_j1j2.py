import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.hamiltonians import J1J2Spec
from paper_2601_20782_b200.lattice import LatticeSpec, pack_bits
from paper_2601_20782_b200.rng import derive_key
spec = J1J2Spec(LatticeSpec.square(10), 1.0, 0.5, marshall=True)
p = rbm.random_parameters(100, 1, derive_key(3, "init"), 0.05)
kern = vmc._energy_kernel(spec, rbm.log_psi_evaluator(p))
rng = np.random.default_rng(0)
bits = np.zeros((65536, 100), dtype=np.uint8)
idx = np.argsort(rng.random((65536, 100)), axis=1)[:, :50]
np.put_along_axis(bits, idx, 1, axis=1)
packed = torch.from_numpy(pack_bits(bits)).cuda()
for _ in range(2): kern.packed(packed)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): kern.packed(packed)
b.record(); torch.cuda.synchronize()
print("j1j2 a1: %.3f ms" % (a.elapsed_time(b) / 5))
