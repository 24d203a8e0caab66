"""Print the GEMM plans (cluster size / clusters) chosen for the C2 shapes (diagnostics)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402
lib = gh.lib()
for c in (1, 2, 4, 8):
    us = C.c_float()
    L.check(lib.gh_debug_gemm_bench(4096, 4096, 64, 8, 0, c, 2, C.byref(us)))
