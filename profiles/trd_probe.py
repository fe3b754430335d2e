"""Phase timing of the tridiagonal reduction (ATK_TRD_PROFILE=1 prints cycles per warp)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

import os  # noqa: E402

ctx = atucker.Context(0)
if "TRD_TILES" in os.environ:  # reduction kernel variant (option trd_tiles)
    ctx.set_option("trd_tiles", int(os.environ["TRD_TILES"]))
for n in [int(a) for a in sys.argv[1:]] or [80, 128, 200]:
    a = np.random.default_rng(n).standard_normal((n, 3 * n))
    s = a @ a.T
    for _ in range(2):
        atucker.sym_eig_top_r(s, max(1, n // 4), ctx=ctx)
