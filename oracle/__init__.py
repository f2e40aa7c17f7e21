"""CPU oracle for the macrofacet hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference algorithm
(`/root/reference/pkg/src/macrofacet`, cited per function as
`<module>.py:<line>`).  It exists for exactly three consumers:

* `tests/` -- the checker the CUDA path is compared against;
* `__graft_entry__.smoke()` -- one tiny cross-check on cuda:0;
* `bench.py` -- the `cpu_baseline` leg and `--impl reference` arm.

Nothing under `paper_2603_00280_b200/` imports it; the product path has
no CPU fallback and fails loudly without its CUDA library.

Pinning: `tests/test_oracle_golden.py` checks this restatement against the
reference test-suite's golden values (test_ndf.py / test_medium.py) and
against fixtures produced by running the reference itself in the build
container (`tests/golden/make_golden.py`, committed with its outputs), so
the oracle is pinned both to the reference's own known-answer vectors and
to the reference's outputs on identical inputs (including bit-identical
SplitMix64 streams and renders).
"""
