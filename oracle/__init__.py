"""TEST INFRASTRUCTURE ONLY — CPU float64 oracle for the AcceRL trainer hot path.

Nothing in the product package (`paper_2603_18464_b200`) imports this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may use it, and only as the checker
or as the timed CPU reference — never as the measured or shipped path.

Parity is pinned: `tests/golden/make_golden.py` imports the real reference
(`/root/reference/pkg/src/asyncrl`) in the build container and writes the
fixtures under `tests/golden/`; `tests/test_oracle.py` checks this
restatement against them and against the reference's own known-answer
values.
"""
