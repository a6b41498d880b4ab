"""Oracle: a plain, slow, obviously correct CPU implementation of slide-wise
Omni-Seg prediction (arxiv 2305.14566), written from PAPER.md and the readings
in DESIGN.md §2.

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it. It shares no code with the
CUDA path (paper_2305_14566_b200) and never imports it.

Pins (tests/test_oracle_*.py, -m "not gpu"): brute-force convolution, SciPy
median filter, textbook Otsu with exact rationals, SPEC worked examples
(tests/golden/), tile-grid closed forms, stitch closed forms, special-weight
closed forms of the network and head (constant network, hand-set theta, the
shift-identity network whose trunk reduces to a per-pixel formula). Parity
unpinned: the end-to-end output of a random network has no closed form; it is
pinned through its parts and those special networks.
"""
from . import frontend, net, pipeline  # noqa: F401
