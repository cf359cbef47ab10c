"""Metropolis–Hastings chain ensemble on the B200 (mirror of the reference
sampler.py:24-251: ``Proposal``, ``pair_table``, ``ChainEnsemble``,
``run_chains``, ``default_chain_count``).

The ensemble state (packed configurations, cached log p, per-chain accepted
counts) lives on the device.  ``step``/``run_steps``/``run_sweeps``/``collect``
launch the fused sweep kernel (csrc/sweep.cuh) for any number of proposals,
with draws from the reference's own counter-based splitmix64 streams, so a run
reproduces the reference ChainEnsemble's decisions (bit for bit in
PER_OPERATION mode; up to documented near-threshold ties in f32/f64).

Sharding: ``chain_offset`` / ``n_chains_total`` place this ensemble's chains at
global ids [offset, offset + n_chains); draws depend on global ids only, so the
shards of a multi-GPU run reproduce the single-GPU run exactly.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import EvaluationFailureError
from .lattice import unpack_bits
from .rng import derive_key, mix64, uniform_from_bits

DEFAULT_SAMPLES_PER_CHAIN = 4
MAX_STEPS_PER_LAUNCH = 1 << 16  # bounded kernel duration


@dataclass(frozen=True)
class Proposal:
    """Single-flip or exchange proposal family (sampler.py:24-39)."""

    kind: str
    sector_weight: int | None = None

    def __post_init__(self):
        if self.kind not in ("flip", "exchange"):
            raise ValueError(f"unknown proposal kind {self.kind!r}")

    @property
    def code(self) -> int:
        return nat.PROPOSAL_FLIP if self.kind == "flip" else nat.PROPOSAL_EXCHANGE


def pair_table(n: int) -> np.ndarray:
    """All unordered site pairs (i < j) in lexicographic order (sampler.py:42-45)."""
    i, j = np.triu_indices(n, k=1)
    return np.stack([i, j], axis=1).astype(np.int64).reshape(-1, 2)


def default_chain_count(n_samples: int) -> int:
    return max(1, n_samples // DEFAULT_SAMPLES_PER_CHAIN)


class TableLogProb:
    """Evaluator backed by a dense table of (unnormalised) log-probabilities
    indexed by configuration code (ref: sampler.py:254-268 table_log_prob);
    the table lives on the device and ChainEnsemble runs mpv_table_sweep.
    Callable on uint8 rows like the reference evaluator."""

    MAX_SITES = 30

    def __init__(self, log_values, n_sites: int, device=None):
        import torch

        nat.require_cuda()
        table = np.asarray(log_values, dtype=np.float64).reshape(-1)
        if table.size != 1 << int(n_sites):
            raise ValueError("table size must be 2^n")
        if not 1 <= int(n_sites) <= self.MAX_SITES:
            raise ValueError(f"table evaluators support 1..{self.MAX_SITES} sites")
        self.n_visible = int(n_sites)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.table = torch.from_numpy(np.ascontiguousarray(table)).to(self.device)

    def __call__(self, bits):
        import torch

        bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
        if bits.shape[1] != self.n_visible:
            raise ValueError("bit matrix width differs from the table's site count")
        rows = torch.from_numpy(bits).to(self.device).to(torch.int64)
        codes = (rows << torch.arange(self.n_visible, device=self.device)).sum(dim=1)
        return self.table[codes].cpu().numpy()


def table_log_prob(log_values, n_sites: int) -> TableLogProb:
    return TableLogProb(log_values, n_sites)


def uniform_log_prob(n_sites: int) -> TableLogProb:
    return TableLogProb(np.zeros(1 << n_sites), n_sites)


def _device_evaluator(evaluator):
    from .rbm import LogProbEvaluator
    from .rescnn import ResCnnEvaluator

    if isinstance(evaluator, ResCnnEvaluator) and evaluator.blob is None:
        raise TypeError("ChainEnsemble fuses the ResCNN tensor-core evaluator (f16 / bf16), not the f64 forward")
    if not isinstance(evaluator, (LogProbEvaluator, TableLogProb, ResCnnEvaluator)):
        raise TypeError(
            f"ChainEnsemble needs a device evaluator (rbm.log_prob_evaluator, sampler.table_log_prob), got "
            f"{type(evaluator).__name__} (the B200 path has no host-callable fallback)")
    return evaluator


class ChainEnsemble:
    """A batch of independent MH chains sharing one device evaluator
    (sampler.py:48-167).  Acceptance counters cover every proposal since the
    last reset."""

    def __init__(self, n_chains, n_sites, proposal: Proposal, evaluator, key, *, chain_offset: int = 0,
                 n_chains_total: int | None = None):
        import torch

        nat.require_cuda()
        self.n_chains = int(n_chains)
        self.n_sites = int(n_sites)
        if self.n_chains < 0 or self.n_sites < 1:
            raise ValueError("need n_chains >= 0 and n_sites >= 1")
        self.proposal = proposal
        self.key = int(np.uint64(key))
        self.chain_offset = int(chain_offset)
        self.n_chains_total = int(n_chains_total) if n_chains_total is not None else self.n_chains + self.chain_offset
        self._evaluator = _device_evaluator(evaluator)
        if self._evaluator.n_visible != self.n_sites:
            raise ValueError("evaluator and ensemble disagree on the number of sites")
        self.device = self._evaluator.device
        self.words = (self.n_sites + 31) // 32
        dev = self.device
        self._bits = torch.zeros((self.n_chains, self.words), dtype=torch.int32, device=dev)
        self._logp = torch.zeros(self.n_chains, dtype=torch.float64, device=dev)
        self._acc = torch.zeros(self.n_chains, dtype=torch.int64, device=dev)
        self._status = torch.tensor([0, 2**63 - 1], dtype=torch.int64, device=dev)
        self._acc_total = torch.zeros(1, dtype=torch.int64, device=dev)
        self.proposed = 0
        self.steps_done = 0
        if proposal.kind == "flip":
            weight = 0
            self.init_draws = self.n_sites
        else:
            weight = self.n_sites // 2 if proposal.sector_weight is None else int(proposal.sector_weight)
            if not 0 <= weight <= self.n_sites:
                raise ValueError(f"sector weight {weight} out of range")
            self.init_draws = self.n_sites - 1
        self._scratch = None
        self._chains = nat.Chains(self.n_chains, self.chain_offset, self.n_sites, self.words,
                                  self._bits.data_ptr(), self._logp.data_ptr(), self._acc.data_ptr(),
                                  self._status.data_ptr(), None, 0)
        self._bind_scratch()
        nat.call("mpv_chains_init", ctypes.byref(self._chains), self.key, proposal.code, weight, self._stream())
        self._launch(0)  # cached log p of the initial configurations (sampler.py:63)
        self._check()

    # -- internals ----------------------------------------------------------
    def _bind_scratch(self):
        from .rescnn import ResCnnEvaluator

        if isinstance(self._evaluator, TableLogProb):
            return
        if isinstance(self._evaluator, ResCnnEvaluator):  # compacted exchange steps
            need = nat.load().mpv_rescnn_mh_scratch_bytes(self.n_chains)
        else:
            need = nat.load().mpv_sweep_scratch_bytes(ctypes.byref(self._snapshot().struct), self.n_chains)
        if self._scratch is None or self._scratch.numel() < need:
            import torch

            self._scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._chains.scratch = self._scratch.data_ptr()
            self._chains.scratch_bytes = self._scratch.numel()

    def _snapshot(self):
        """The evaluator's snapshot in this ensemble's sweep layout (exchange: one
        chain per warp, DeviceSnapshot.for_proposal)."""
        return self._evaluator.snapshot.for_proposal(self.proposal.kind)

    @property
    def layout_label(self) -> str:
        """Format / arithmetic / accumulator / lane layout of this ensemble's sweep."""
        from .rescnn import ResCnnEvaluator

        if isinstance(self._evaluator, (TableLogProb, ResCnnEvaluator)):
            return type(self._evaluator).__name__
        return self._snapshot().label

    def _stream(self):
        return nat.stream_handle(self.device)

    def _launch(self, n_steps, thin=0, samples=None, n_samples_total=0, round_offset=0, row0=0):
        self._refresh_pending = False  # every launch refreshes the cached log p from the bits first
        sp = samples.data_ptr() if samples is not None else None
        from .rescnn import ResCnnEvaluator

        if isinstance(self._evaluator, ResCnnEvaluator):
            ev = self._evaluator
            nat.call("mpv_rescnn_mh_sweep", ev.L, ev.n_res, ev.fmt.code, ev.blob.data_ptr(), ctypes.byref(self._chains),
                     self.key, self.proposal.code, self.init_draws, self.steps_done, int(n_steps), int(thin), sp,
                     int(n_samples_total), self.n_chains_total, int(round_offset), int(row0), self._stream())
        elif isinstance(self._evaluator, TableLogProb):
            nat.call("mpv_table_sweep", self._evaluator.table.data_ptr(), ctypes.byref(self._chains), self.key,
                     self.proposal.code, self.init_draws, self.steps_done, int(n_steps), int(thin), sp,
                     int(n_samples_total), self.n_chains_total, int(round_offset), int(row0), self._stream())
        else:
            nat.call("mpv_mh_sweep", ctypes.byref(self._snapshot().struct), ctypes.byref(self._chains),
                     self.key, self.proposal.code, self.init_draws, self.steps_done, int(n_steps), int(thin), sp,
                     int(n_samples_total), self.n_chains_total, int(round_offset), int(row0), self._stream())
        self.steps_done += int(n_steps)
        self.proposed += self.n_chains * int(n_steps)

    def _check(self, st=None):
        """Raise the first recorded evaluation failure.  The status words are
        sticky (first non-finite (step, chain)), so a check after several
        unchecked launches reports the same failure as immediate checking."""
        if st is None:
            self._flush_refresh()
            st = self._status.cpu().numpy()
        if st[0] != 0:
            key = int(st[1])
            step, chain = key >> 32, key & 0xFFFFFFFF
            bits = self._proposal_bits(chain, step)
            raise EvaluationFailureError(
                f"non-finite log probability for configuration bits {bits.tolist()}",
                context={"bits": bits, "chain": self.chain_offset + chain, "step": step})

    def _proposal_bits(self, chain, step):
        """Configuration whose evaluation failed: the chain is frozen at the
        state before `step`; step 0 is the initial evaluation."""
        x = unpack_bits(self._bits[chain:chain + 1].cpu().numpy().view(np.uint32), self.n_sites)[0].copy()
        if step == 0:
            return x
        g = 0x9E3779B97F4A7C15
        s0 = mix64(self.key ^ (((self.chain_offset + chain + 1) * g) & 0xFFFFFFFFFFFFFFFF))
        t = self.init_draws + 2 * (step - 1)
        u = float(uniform_from_bits(np.uint64(mix64((s0 + (t + 1) * g) & 0xFFFFFFFFFFFFFFFF))))
        if self.proposal.kind == "flip":
            x[int(u * self.n_sites)] ^= 1
        else:
            i, j = pair_table(self.n_sites)[int(u * (self.n_sites * (self.n_sites - 1) // 2))]
            x[i], x[j] = x[j], x[i]
        return x

    # -- reference API ------------------------------------------------------
    def set_evaluator(self, evaluator, check: bool = True):
        """Swap the target; refreshes every chain's cached log-probability
        (sampler.py:90-93).  check=False defers both the refresh and the failure
        check: every sweep launch recomputes the cached log p from the bits at
        its start, so the refresh rides on the next launch (a zero-step launch
        runs first only if log_probs / state is read before any sweep), and a
        non-finite refreshed value is reported by the next checked call with
        step 0, as an immediate check would."""
        ev = _device_evaluator(evaluator)
        if ev.n_visible != self.n_sites:
            raise ValueError("evaluator and ensemble disagree on the number of sites")
        self._evaluator = ev
        self._bind_scratch()
        if check:
            self._launch(0)
            self._check()
        else:
            self._refresh_pending = True

    def _flush_refresh(self):
        if getattr(self, "_refresh_pending", False):
            self._launch(0)

    def reset_counters(self):
        self._acc.zero_()
        self.proposed = 0

    @property
    def evaluator(self):
        return self._evaluator

    # -- checkpoint / resume (beyond the reference, which has none: SURVEY §5) --
    def state_dict(self) -> dict:
        """Everything that determines the continuation: packed configurations,
        cached log p, per-chain acceptance counters, the draw counter
        (steps_done) and the stream key / proposal / shard.  The theta
        accumulators are a function of the bits (refreshed at every launch),
        so they are not stored."""
        self._flush_refresh()
        self._check()
        return {"format": "mpv-chains-v1", "n_sites": self.n_sites, "n_chains": self.n_chains,
                "chain_offset": self.chain_offset, "n_chains_total": self.n_chains_total, "key": self.key,
                "proposal": self.proposal.kind, "sector_weight": self.proposal.sector_weight,
                "init_draws": self.init_draws, "steps_done": self.steps_done, "proposed": self.proposed,
                "bits": self._bits.cpu().numpy().copy(), "log_probs": self._logp.cpu().numpy().copy(),
                "accepted": self._acc.cpu().numpy().copy()}

    def load_state_dict(self, state: dict):
        """Resume from state_dict(): the continuation is bit-identical to an
        uninterrupted run (draws depend only on (key, chain, draw counter))."""
        import torch

        if state.get("format") != "mpv-chains-v1":
            raise ValueError("not an mpv-chains-v1 state")
        for k in ("n_sites", "n_chains", "chain_offset", "n_chains_total", "key", "init_draws"):
            if int(state[k]) != int(getattr(self, k)):
                raise ValueError(f"state mismatch in {k}: {state[k]} vs {getattr(self, k)}")
        if state["proposal"] != self.proposal.kind:
            raise ValueError("state was recorded with a different proposal")
        self._bits.copy_(torch.from_numpy(np.asarray(state["bits"], dtype=np.int32)))
        self._logp.copy_(torch.from_numpy(np.asarray(state["log_probs"], dtype=np.float64)))
        self._acc.copy_(torch.from_numpy(np.asarray(state["accepted"], dtype=np.int64)))
        self.steps_done = int(state["steps_done"])
        self.proposed = int(state["proposed"])

    def save_state(self, path):
        st = self.state_dict()
        np.savez(path, **{k: np.asarray(v) if not isinstance(v, str) else np.array(v) for k, v in st.items()
                          if v is not None}, has_weight=np.array(st["sector_weight"] is not None))
        return path

    def load_state(self, path):
        with np.load(path, allow_pickle=False) as z:
            st = {k: z[k] for k in z.files}
        st = {k: (str(v) if v.dtype.kind == "U" else (v if v.ndim else v.item())) for k, v in st.items()}
        st.setdefault("sector_weight", None)
        self.load_state_dict(st)

    @property
    def bits(self) -> np.ndarray:
        return unpack_bits(self._bits.cpu().numpy().view(np.uint32), self.n_sites)

    @property
    def packed_bits(self):
        """Device tensor of packed configurations (int32 view of uint32 words)."""
        return self._bits

    @property
    def log_probs(self) -> np.ndarray:
        self._flush_refresh()
        return self._logp.cpu().numpy().copy()

    @property
    def accepted(self) -> int:
        nat.call("mpv_sum_i64", self._acc.data_ptr(), self.n_chains, self._acc_total.data_ptr(), self._stream())
        return int(self._acc_total.item())

    @property
    def accepted_per_chain(self):
        return self._acc

    @property
    def acceptance_rate(self) -> float:
        return self.accepted / self.proposed if self.proposed else float("nan")

    def step(self):
        """One MH proposal per chain (sampler.py:111-133)."""
        self.run_steps(1)

    def run_steps(self, n_steps: int, check: bool = True):
        remaining = int(n_steps)
        while remaining > 0:
            chunk = min(remaining, MAX_STEPS_PER_LAUNCH)
            self._launch(chunk)
            remaining -= chunk
        if check:
            self._check()

    def run_sweeps(self, n_sweeps: int, check: bool = True):
        self.run_steps(int(n_sweeps) * self.n_sites, check)

    def collect_packed(self, n_samples: int, thin_steps: int = 1, check: bool = True):
        """collect() leaving the samples on the device as packed uint32 words
        [rows of this shard, words] (int32 tensor)."""
        import torch

        n_samples, thin_steps = int(n_samples), int(thin_steps)
        if thin_steps < 1:
            raise ValueError("thin_steps must be >= 1")
        base, extra = divmod(n_samples, self.n_chains_total)
        rounds = base + (1 if extra else 0) if n_samples else 0
        first = self.chain_offset
        last = self.chain_offset + self.n_chains
        row0 = first * base + min(first, extra)
        row1 = last * base + min(last, extra)
        samples = torch.zeros((row1 - row0, self.words), dtype=torch.int32, device=self.device)
        r = 0
        per_launch = max(1, MAX_STEPS_PER_LAUNCH // thin_steps)
        while r < rounds:
            k = min(per_launch, rounds - r)
            self._launch(k * thin_steps, thin_steps, samples, n_samples, r, row0)
            r += k
        if check:
            self._check()
        return samples

    def collect(self, n_samples: int, thin_steps: int = 1) -> np.ndarray:
        """Record n_samples total, thinned by proposal steps, merged chain-major
        (sampler.py:142-167); returns this shard's uint8 rows."""
        import torch

        packed = self.collect_packed(n_samples, thin_steps, check=False)
        out = torch.empty((packed.shape[0], self.n_sites), dtype=torch.uint8, device=self.device)
        if packed.shape[0]:
            nat.call("mpv_unpack_bits", packed.data_ptr(), packed.shape[0], self.n_sites, out.data_ptr(),
                     self._stream())
        # fresh pinned block from torch's caching host allocator (no host memcpy):
        # the returned array keeps it alive, and device_pack() re-uploads it by DMA.
        # The status words ride along: one synchronisation for samples + check.
        host = torch.empty(out.shape, dtype=torch.uint8, pin_memory=True)
        st = torch.empty(2, dtype=torch.int64, pin_memory=True)
        host.copy_(out, non_blocking=True)
        st.copy_(self._status, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        self._check(st.numpy())
        return host.numpy()


def run_chains(n_chains, n_samples, burn_in_steps, thin_steps, seed, logprob, proposal: Proposal, n_sites):
    """Run independent chains and pool samples (sampler.py:221-247)."""
    if min(n_chains, n_samples) < 1 or thin_steps < 1 or burn_in_steps < 0:
        raise ValueError("counts must be positive")
    ensemble = ChainEnsemble(n_chains, n_sites, proposal, logprob, derive_key(seed, "chains"))
    ensemble.run_steps(burn_in_steps)
    ensemble.reset_counters()
    samples = ensemble.collect(n_samples, thin_steps)
    return samples, ensemble.acceptance_rate
