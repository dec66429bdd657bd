"""CPU oracle for the LiveCap pose + non-rigid Gauss-Newton hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package, and only as the checker or the timed CPU baseline -- never as the
thing measured or shipped.  The product (`paper_1810_02648_b200`) never
imports it and fails loudly when its CUDA library is missing.

What it is: a numpy (+ a small C file for the two numba kernels) restatement
of the reference `montrack` package's hot path,
each function citing the reference file:line it follows.  Reference paths
are relative to `/root/reference/pkg/src/montrack/`.

How it is pinned: `tools/make_golden.py` runs the real reference (importable
in the build container only) on small seeded scenes and commits the inputs and
outputs under `tests/golden/`; `tests/test_oracle_golden.py` checks this
oracle against them (bit-exact for integer/index outputs, tight fp64
tolerances for energies and positions).
"""
