"""CPU oracle for the hybridbench hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithms (arXiv 1303.2171's
`hybridbench`, /root/reference/pkg/src/hybridbench/) for the five
work-partitioned kernels and their input generators.  Every function cites
the reference file:line it follows.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports the reference package
in the dev container and writes tests/golden/*.npz) and against the
reference's own known-answer tests (splitmix64 seed-0 KAT,
tests/test_datasets.py:20-25; SpMV perm/split KATs,
tests/test_kernels_irregular.py:70-89; LUT KATs,
tests/test_kernels_regular.py:184-193).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package, and only as the checker or
the timed CPU baseline — never as the product path.  The product package
(paper_1303_2171_b200) does not import it.
"""
