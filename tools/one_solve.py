"""One single-grid solve (for ncu source-level profiling): python tools/one_solve.py redrec 256 153 257"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06182_b200 import load_native  # noqa: E402
from paper_2504_06182_b200.inputs import sample_grids  # noqa: E402

solver, n, hp, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4], 0)
k = round(0.6 * n * n)
lib = load_native()
occ = sample_grids(seed, 1, n, n, k)
for _ in range(2):
    r = lib.grid_solve(solver, occ, n, n, hp)
print(solver, n, hp, len(r.path_src), r.total_displacement)
