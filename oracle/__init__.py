"""CPU oracle for the ME-Switch multi-expert serving hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2406_09041_b200/`) imports this directory.  Only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` may import it, and only as the checker (or as the timed reference
CPU arm), never as the thing measured for the GPU arm.

Every function restates the reference algorithm in plain numpy and cites the
reference file:line it follows (`/root/reference/pkg/src/meswitch/*.py`,
`/root/reference/SPEC.md`).  The restatement is pinned against the real
reference by the golden fixtures under `tests/golden/` (generated in the build
container by `tests/golden/make_golden.py`, which imports the reference
package) -- see `tests/test_oracle_golden.py`.
"""
