"""Multi-process (gloo, world size 2, CPU) coverage of the chain-sharding
host logic: shard/row ranges reproduce the single-process layout, and the
all-reduced statistics equal the single-process reference estimators."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_20782_b200 import parallel

N_CHAINS, N_SAMPLES = 37, 150


def _fake_eps(n_samples):
    return np.random.default_rng(5).normal(3.0, 2.0, n_samples)


def reference_stats():
    eps = _fake_eps(N_SAMPLES)
    base, extra = divmod(N_SAMPLES, N_CHAINS)
    counts = np.array([base + (1 if c < extra else 0) for c in range(N_CHAINS)])
    ids = np.repeat(np.arange(N_CHAINS), counts)
    means = np.bincount(ids, weights=eps, minlength=N_CHAINS) / counts
    err = float(np.sqrt(means.var(ddof=1) / means.size))  # vmc.mc_error of chain means
    return float(eps.mean()), err


def _worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    off, cnt = parallel.shard(N_CHAINS, rank, world)
    r0, r1 = parallel.sample_rows(N_SAMPLES, N_CHAINS, off, cnt)
    eps = torch.from_numpy(_fake_eps(N_SAMPLES)[r0:r1].copy())
    counts = parallel.chain_counts(N_SAMPLES, N_CHAINS, off, cnt)
    stats = parallel.energy_statistics(eps, counts, accepted=10 * (rank + 1), proposed=100)
    q.put((rank, off, cnt, r0, r1, stats))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_layout_single_process():
    for world in (1, 2, 3, 8):
        offs = [parallel.shard(N_CHAINS, r, world) for r in range(world)]
        assert sum(c for _, c in offs) == N_CHAINS
        rows = [parallel.sample_rows(N_SAMPLES, N_CHAINS, o, c) for o, c in offs]
        assert rows[0][0] == 0 and rows[-1][1] == N_SAMPLES
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))


@pytest.mark.timeout(120)
def test_gloo_world2_statistics():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    energy, err = reference_stats()
    for rank, off, cnt, r0, r1, stats in results:
        assert stats["energy"] == pytest.approx(energy, rel=1e-12)
        assert stats["mc_error"] == pytest.approx(err, rel=1e-9)
        assert stats["acceptance"] == pytest.approx(30 / 200)
        assert stats["n_chains"] == N_CHAINS and stats["n_samples"] == N_SAMPLES
    assert results[0][3] == 0 and results[0][4] == results[1][3] and results[1][4] == N_SAMPLES


def _stats_worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    o, eps, w = _fake_vmc()
    half = o.shape[0] // 2
    sl = slice(0, half) if rank == 0 else slice(half, None)
    f, s, e = parallel.sharded_statistics(o[sl], eps[sl], w[sl])
    q.put((rank, f.numpy(), s.numpy(), float(e)))
    dist.destroy_process_group()


def _fake_vmc():
    rng = np.random.default_rng(11)
    o = torch.from_numpy(rng.normal(size=(40, 6)) + 1j * rng.normal(size=(40, 6)))
    eps = torch.from_numpy(rng.normal(size=40) + 1j * rng.normal(size=40))
    w = torch.from_numpy(rng.random(40))
    w = w / w.sum()
    return o, eps, w


@pytest.mark.timeout(120)
def test_gloo_sharded_forces_and_s_matrix():
    """Two ranks holding halves of the samples reproduce the single-process
    weighted forces and S-matrix (ref vmc.py:145-188)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stats_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    o, eps, w = _fake_vmc()
    oc = np.conj(o.numpy())
    wn, en = w.numpy(), eps.numpy()
    f_ref = (oc * wn[:, None]).T @ en - (wn @ oc) * (wn @ en)
    mean = wn @ o.numpy()
    c = o.numpy() - mean[None, :]
    s_ref = np.conj(c).T @ (c * wn[:, None])
    s_ref = 0.5 * (s_ref + np.conj(s_ref).T)
    for _, f, s, e in res:
        assert np.allclose(f, f_ref, atol=1e-13)
        assert np.allclose(s, s_ref, atol=1e-13)
        assert e == pytest.approx(float((wn @ en).real), abs=1e-14)
