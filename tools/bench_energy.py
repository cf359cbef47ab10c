"""Time the f64 local-energy kernel alone at the bench workload (10x10 TFIM, alpha=2, 65536 samples)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec, HeisenbergSpec
from paper_2601_20782_b200.lattice import LatticeSpec, pack_bits
from paper_2601_20782_b200.rng import derive_key
for name, spec, alpha in (("tfim10x10 a2", TfimSpec(LatticeSpec.square(10), 1.0, 3.04), 2),
                          ("heis10x10 a4", HeisenbergSpec(LatticeSpec.square(10), 1.0), 4)):
    p = rbm.random_parameters(100, alpha, derive_key(0, "init"), 0.01)
    psi = rbm.log_psi_evaluator(p)
    kern = vmc._energy_kernel(spec, psi)
    if len(sys.argv) > 1 and sys.argv[1] not in name:
        continue
    bits = np.random.default_rng(0).integers(0, 2, size=(65536, 100), dtype=np.uint8)
    packed = torch.from_numpy(pack_bits(bits)).cuda()
    try:
        for _ in range(3):
            kern.packed(packed)
    except ValueError as exc:
        print(f"{name}: {exc}")
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        kern.packed(packed)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    terms = 100 if isinstance(spec, TfimSpec) else 200
    print(f"{name}: {ms:.3f} ms  ({65536/ms*1e3:.3e} samples/s, {65536*terms*p.n_hidden*10/ms/1e9:.2f} TFLOP64/s algorithmic)")
