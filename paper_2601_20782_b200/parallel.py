"""Chain sharding across GPUs (one process per GPU, torch.distributed).

Chains are independent MH chains whose draws depend only on (key, global
chain id) (ref rng.py:63-77; pinned by the reference's
tests/test_rng.py:33-39), so rank r simply owns the contiguous global ids
[offset_r, offset_r + count_r).  Samples stay where they are drawn; the only
collectives are the per-iteration all-reduces of energy sums, split-chain
moments and acceptance counts (NCCL on GPUs, gloo on CPU for the tests).
Concatenating the ranks' sample rows in rank order reproduces the
single-process chain-major sample matrix (ref sampler.py:152-166) exactly.
"""
from __future__ import annotations

import math

import numpy as np


def shard(n_total: int, rank: int, world: int):
    """(offset, count) of rank's contiguous slice of n_total chains."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n_total), int(world))
    offset = rank * base + min(rank, extra)
    return offset, base + (1 if rank < extra else 0)


def sample_rows(n_samples: int, n_chains_total: int, offset: int, count: int):
    """Rows [row0, row1) of the chain-major sample matrix owned by chains
    [offset, offset+count) (chain c owns floor(S/C) + [c < S mod C] rows)."""
    base, extra = divmod(int(n_samples), int(n_chains_total))
    row = lambda c: c * base + min(c, extra)  # noqa: E731
    return row(offset), row(offset + count)


def chain_counts(n_samples: int, n_chains_total: int, offset: int, count: int) -> np.ndarray:
    base, extra = divmod(int(n_samples), int(n_chains_total))
    ids = np.arange(offset, offset + count)
    return base + (ids < extra).astype(np.int64)


def all_reduce_sum(values, group=None):
    """SUM all-reduce of a float64 vector across ranks (identity without a
    process group).  `values` is a torch tensor on the rank's device."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values


def energy_statistics(eps_real, counts, accepted, proposed, group=None):
    """Global energy mean, split-chain MC error and acceptance from one rank's
    shard (ref vmc.py:592-604, sampler.py:107-109).

    eps_real: this rank's sample energies (chain-major rows, torch f64 tensor);
    counts: samples per local chain (numpy int); accepted/proposed: local totals.
    The split-chain error uses the all-reduced moments of the per-chain means
    (sum m, sum m^2, number of chains): var = (sum m^2 - (sum m)^2 / C) / (C - 1).
    """
    import torch

    dev = eps_real.device
    cnt = torch.as_tensor(np.asarray(counts), device=dev)
    chain_ids = torch.repeat_interleave(torch.arange(len(counts), device=dev), cnt)
    sums = torch.zeros(len(counts), dtype=torch.float64, device=dev).index_add_(0, chain_ids, eps_real)
    means = sums / cnt.to(torch.float64)
    red = torch.stack([
        eps_real.sum(), torch.tensor(float(eps_real.numel()), dtype=torch.float64, device=dev),
        means.sum(), (means * means).sum(), torch.tensor(float(len(counts)), dtype=torch.float64, device=dev),
        torch.tensor(float(accepted), dtype=torch.float64, device=dev),
        torch.tensor(float(proposed), dtype=torch.float64, device=dev)])
    all_reduce_sum(red, group)
    e_sum, n, m1, m2, c, acc, prop = (float(v) for v in red.cpu())
    var = max(m2 - m1 * m1 / c, 0.0) / (c - 1) if c > 1 else float("nan")
    return {"energy": e_sum / n, "mc_error": math.sqrt(var / c) if c > 1 else float("nan"),
            "acceptance": acc / prop if prop else float("nan"), "n_samples": int(n), "n_chains": int(c)}


def sharded_ensemble(n_chains_total, n_sites, proposal, evaluator, key, rank, world):
    """This rank's ChainEnsemble over its slice of global chain ids."""
    from .sampler import ChainEnsemble

    offset, count = shard(n_chains_total, rank, world)
    return ChainEnsemble(count, n_sites, proposal, evaluator, key, chain_offset=offset,
                         n_chains_total=n_chains_total)


def sharded_statistics(o, eps, weights, group=None):
    """Forces and S-matrix of the reference estimators (vmc.py:145-188) from
    per-rank shards of the sample set, with NCCL/gloo all-reduces only:

      F = sum_w conj(O) eps - (sum_w conj O)(sum_w eps)
      S = sum_w (O - Obar)^H (O - Obar),  Obar = sum_w O     (two passes)

    `weights` are this rank's sample weights normalised over the GLOBAL sample
    count, so the all-reduced sums are the single-process weighted sums.
    Returns (f, s, energy) identical on every rank (then every rank solves the
    same SR system and keeps identical parameters)."""
    import torch

    w = weights.to(o.dtype)
    oc = o.conj()
    s_oe = (oc * w[:, None]).T @ eps
    s_o = w @ oc
    s_e = (w @ eps).reshape(1)
    s_wo = w @ o
    first = torch.cat([s_oe, s_o, s_e, s_wo])
    all_reduce_sum(first, group)
    P = o.shape[1]
    s_oe, s_o, s_e, mean = first[:P], first[P:2 * P], first[2 * P], first[2 * P + 1:]
    f = s_oe - s_o * s_e
    c = o - mean[None, :]
    s = c.conj().T @ (c * w[:, None])
    all_reduce_sum(s, group)
    s = 0.5 * (s + s.conj().T)
    return f, s, s_e.real
