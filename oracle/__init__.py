"""TEST INFRASTRUCTURE ONLY — CPU oracle for the B200 hot path.

This package restates, in plain numpy, the reference (flowbench 0.1.0,
arXiv 1910.03032) algorithms on the hot path so the CUDA path can be checked
on the GPU box, where /root/reference does not exist.  Each function cites
the reference file:line it follows.  It is pinned against golden vectors
produced by the real reference (tests/golden/make_golden.py) in the CPU test
suite (tests/test_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline.  The product package (paper_1910_03032_b200) never imports
it.
"""
