"""Two ranks (gloo, both on cuda:0 — no kernel waits on another rank) run the
sharded training loop and reproduce the single-process run: same samples
(global chain ids), all-reduced forces / S / energy / error / acceptance."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(solver="dense"):
    if solver == "exact":
        from paper_2601_20782_b200 import vmc
        from paper_2601_20782_b200.hamiltonians import TfimSpec
        from paper_2601_20782_b200.lattice import LatticeSpec

        return vmc.TrainConfig(TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=4, n_samples=256, eta=0.02, seed=3,
                               sampling_mode="exact")
    from paper_2601_20782_b200 import F32, vmc
    from paper_2601_20782_b200.hamiltonians import TfimSpec
    from paper_2601_20782_b200.lattice import LatticeSpec

    return vmc.TrainConfig(TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=4, n_samples=256, n_chains=64,
                           eta=0.02, seed=3, sampling_format=F32, sr_solver=solver, cg_tol=1e-12)


def _worker(rank, world, port, q, solver):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_20782_b200 import vmc

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = vmc.train(_cfg(solver))
    q.put((rank, [(r["energy"], r["mc_error"], r["acceptance"], r["sigma_hat"]) for r in res.records],
           res.params.w))
    dist.destroy_process_group()


@pytest.mark.parametrize("solver", ["dense", "cg", "exact", "minsr"])
def test_two_rank_training_matches_single(cuda, solver):
    from paper_2601_20782_b200 import vmc

    single = vmc.train(_cfg(solver))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, solver)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, recs, w in res:
        for (e, err, acc, sig), r in zip(recs, single.records):
            assert e == pytest.approx(r["energy"], rel=1e-10, abs=1e-12)
            assert err == pytest.approx(r["mc_error"], rel=1e-8)
            assert acc == r["acceptance"] or (np.isnan(acc) and np.isnan(r["acceptance"]))
            # sigma-hat pools per-rank unique batches (duplicates across ranks count twice)
            assert sig == pytest.approx(r["sigma_hat"], rel=0.2)
        np.testing.assert_allclose(w, single.params.w, rtol=1e-8, atol=1e-11)
