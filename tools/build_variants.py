"""Build tuning variants of libfiedler.so (tile size / pipeline stages / min blocks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_04386_b200 import build as b  # noqa: E402

VARIANTS = [(2048, 2, 4, 256, 4), (2048, 2, 4, 256, 8), (2048, 2, 4, 256, 6), (2048, 2, 3, 256, 8), (1024, 2, 6, 256, 4), (1024, 3, 5, 256, 8)]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants")
os.makedirs(out, exist_ok=True)
for T, S, M, P, C in VARIANTS:
    name = os.path.join(out, "libfiedler_T%d_S%d_M%d_P%d_C%d.so" % (T, S, M, P, C))
    b.build(defines=("FDL_TILE_T=%d" % T, "FDL_STAGES=%d" % S, "FDL_PASS_MINB=%d" % M,
                     "FDL_PASS_THREADS=%d" % P, "FDL_CHUNK=%d" % C), out=name)
    print(name)
