"""TEST INFRASTRUCTURE ONLY — CPU oracle for the unwrap hot path.

This package is the *checker*: a numpy restatement of the reference
algorithm (`phaseirls`, /root/reference/pkg/src/phaseirls) used by
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py`.  Nothing in `paper_2401_09961_b200/` imports
it; the product path is CUDA-only and fails loudly without its extension.

Parity pinning: `tests/golden/make_golden.py` ran the unmodified reference
in the build container and committed its outputs under `tests/golden/`;
`tests/test_oracle_golden.py` checks this restatement against them.
"""
