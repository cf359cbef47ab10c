"""CPU oracle for the MH-sampling / local-energy hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference CPU algorithm (arXiv 2601.20782, `mpvmc`,
/root/reference/pkg/src/mpvmc) so the CUDA path can be checked against it:

* ``oracle.port``  — ctypes wrapper of ``oracle/c/oracle_port.c`` (plain-C
  restatement of ``_kernels.rounded_forward``/``rounded_log_prob``,
  ``rbm._fast_forward``, ``ChainEnsemble`` and ``vmc.local_energies``);
* ``oracle.rng``   — numpy restatement of ``rng.py`` (splitmix64 streams, key derivation);
* ``oracle.model`` — numpy models: the incremental-f64 sweep ("device model",
  SURVEY §0.11), the native f32-accumulation forward, and the O(N·M) local energies.

Pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports /root/reference in the build container
and commits ``tests/golden/*.npz``); ``tests/test_oracle.py`` checks the pin.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / baseline — never as the
thing measured or shipped.  The product package ``paper_2601_20782_b200`` does
not import it.
"""
