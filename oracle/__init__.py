"""CPU oracle for the cached generation step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import or execute anything in this package, and
only as the checker or the timed CPU baseline. The product package
(paper_1611_09482_b200) never imports it and fails loudly without its CUDA
library instead of falling back here.

Pinning: plain mode (oracle/plain.py) is checked against outputs of the
unmodified reference (tests/golden/plain_reference.npz, oracle/make_golden.py).
The gated cell (oracle/cell.py) has no reference counterpart; it is pinned by
3-way fp64 self-equivalence and constructed-weight cases.
"""
