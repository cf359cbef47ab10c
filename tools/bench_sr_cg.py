"""Time the factored O products of the matrix-free SR at config 2 (U=65536, N=100, M=200)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.rng import derive_key

U, N, alpha = 65536, 100, 2
p = rbm.random_parameters(N, alpha, derive_key(0, "init"), 0.01)
bits = torch.from_numpy(np.random.default_rng(0).integers(0, 2, size=(U, N), dtype=np.uint8)).cuda()
fo = vmc.FactoredLogDerivatives(p, bits)
P = N + p.n_hidden + p.n_hidden * N
v = torch.randn(P, dtype=torch.complex128, device="cuda")
u = torch.randn(U, dtype=torch.complex128, device="cuda")
def tm(f, k=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / k
M = p.n_hidden
vw = v[N + M:].reshape(M, N)
print("o_v   %.3f ms" % tm(lambda: fo.o_v(v)))
print("oh_u  %.3f ms" % tm(lambda: fo.oh_u(u)))
xc = bits.to(torch.complex128)
print("torch zgemm T@vW (reference shape)  %.3f ms" % tm(lambda: fo.t @ vw))
ux = u[:, None] * xc
print("torch zgemm T^H (uX)  %.3f ms" % tm(lambda: fo.t.mH @ ux))
