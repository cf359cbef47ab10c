"""Lockstep decision parity of a device ChainEnsemble against the oracle's
restatement of the reference ChainEnsemble (sampler.py:111-133) with the
per-operation f32 evaluator (_kernels.py:95-129) — test infrastructure.

Both ensembles take the same proposals (same streams, same draw schedule).  A
decision mismatch is accepted only as a near-threshold tie:
at the chain's first divergent step, log u must lie within the two f32
evaluations' error bars around the exact f64 increment,

    |log u - D64| <= 2e-5 max(1, |lp_old|, |lp_new|) + |D_ref - D64| + 1e-6 |log u|

(2e-5: the north-star 1e-5 relative bar on each of the device's two log p;
|D_ref - D64|: the reference's own f32 error at that step).  Every tie is
recorded; the diverged chain is then resynchronised to the reference state and
the comparison continues.  Any other divergence fails.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import port


def _draws(key, chain, t):
    u = port.stream_uniforms(int(key), 1, 2, chain0=int(chain), t0=int(t))
    return float(u[0, 0]), float(u[1, 0])


def run_lockstep(ens, ev, ref, snap_params, params64, n_steps, kind="flip", check_every=100):
    """Advance the device ensemble `ens` (evaluator `ev`) and the oracle
    PortEnsemble `ref` one step at a time.  Returns (ties, log-p error stats)."""
    n = ens.n_sites
    p64 = port.Params(params64.a, params64.b, params64.w)
    psnap = port.Params(snap_params.a, snap_params.b, snap_params.w)
    ties = []
    stats = {"dev_vs_f64": 0.0, "ref_vs_f64": 0.0, "dev_vs_ref": 0.0}
    for s in range(n_steps):
        x_before = ref.bits.copy()
        lp_ref_before = ref.logp.copy()
        lp_dev_before = ens.log_probs
        t = ens.init_draws + 2 * ens.steps_done
        ens.run_steps(1)
        ref.run_steps(1)
        dev_bits = ens.bits
        bad = np.nonzero(np.any(dev_bits != ref.bits, axis=1))[0]
        for c in bad:
            u_sel, u_acc = _draws(ens.key, c, t)
            x_new = x_before[c].copy()
            if kind == "flip":
                x_new[int(u_sel * n)] ^= 1
            else:
                pairs = np.stack(np.triu_indices(n, k=1), axis=1)
                i, j = pairs[int(u_sel * (n * (n - 1) // 2))]
                x_new[i], x_new[j] = x_new[j], x_new[i]
            lp_ref_new = float(port.rounded_log_prob(psnap, x_new[None, :], "f32")[0])
            lp_dev_new = float(ev(x_new[None, :])[0])
            lp64 = port.f64_forward(p64, np.stack([x_before[c], x_new]))[0]
            d_ref = lp_ref_new - float(lp_ref_before[c])
            d_dev = lp_dev_new - float(lp_dev_before[c])
            d64 = float(lp64[1] - lp64[0])
            logu = math.log(u_acc)
            scale = max(1.0, abs(lp64[0]), abs(lp64[1]))
            tol = 2e-5 * scale + abs(d_ref - d64) + 1e-6 * abs(logu)
            rec = {"step": s, "chain": int(c), "log_u": logu, "d_ref": d_ref, "d_dev": d_dev, "d64": d64,
                   "gap": abs(logu - d64), "tol": tol}
            assert abs(logu - d64) <= tol, f"unexplained divergence {rec}"
            assert abs(d_dev - d64) <= 2e-5 * scale, f"device increment outside the f32 bar {rec}"
            ties.append(rec)
        if len(bad):
            # resync: the diverged chains take the reference state
            st = ens.state_dict()
            words = st["bits"].shape[1]
            for c in bad:
                w = np.zeros(words, dtype=np.uint32)
                for k in np.nonzero(ref.bits[c])[0]:
                    w[k >> 5] |= np.uint32(1) << np.uint32(k & 31)
                st["bits"][c] = w.view(np.int32)
            ens.load_state_dict(st)
            ens.set_evaluator(ev)  # refresh the cached log p of the resynchronised chains
        if (s + 1) % check_every == 0 or s + 1 == n_steps:
            # log p bar: the device within 1e-5 max(1, |lp|) of the
            # exact f64 value, and no further from the reference's f32 value than
            # that plus the reference's own f32 error
            lp = ens.log_probs
            lp64 = port.f64_forward(p64, ens.bits)[0]
            scale = np.maximum(1.0, np.abs(lp64))
            dev64 = np.abs(lp - lp64) / scale
            ref64 = np.abs(ref.logp - lp64) / scale
            devref = np.abs(lp - ref.logp) / scale
            assert dev64.max() < 1e-5, f"step {s}: device log p {dev64.max():.2e} from f64"
            assert np.all(devref <= 1e-5 + ref64), f"step {s}: device vs reference beyond the f32 bars"
            stats["dev_vs_f64"] = max(stats["dev_vs_f64"], float(dev64.max()))
            stats["ref_vs_f64"] = max(stats["ref_vs_f64"], float(ref64.max()))
            stats["dev_vs_ref"] = max(stats["dev_vs_ref"], float(devref.max()))
    return ties, stats
