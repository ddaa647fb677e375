"""Build tuning variants of libfiedler.so (tile size / pipeline stages / min blocks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_04386_b200 import build as b  # noqa: E402

VARIANTS = [(2048, 2, 4, 256), (3072, 2, 2, 256), (1536, 2, 5, 256), (4096, 2, 2, 512), (2048, 2, 2, 512), (4096, 2, 1, 1024)]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants")
os.makedirs(out, exist_ok=True)
for T, S, M, P in VARIANTS:
    name = os.path.join(out, "libfiedler_T%d_S%d_M%d_P%d.so" % (T, S, M, P))
    b.build(defines=("FDL_TILE_T=%d" % T, "FDL_STAGES=%d" % S, "FDL_PASS_MINB=%d" % M,
                     "FDL_PASS_THREADS=%d" % P), out=name)
    print(name)
