"""Build tuning variants of libfiedler.so (-D overrides of tuning macros)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_04386_b200 import build as b  # noqa: E402

# usage: python tools/build_variants.py "[dict(FDL_X=1), dict(FDL_X=2)]"
VARIANTS = eval(sys.argv[1]) if len(sys.argv) > 1 else [dict(FDL_HEAVY_DEG=64), dict(FDL_HEAVY_DEG=128)]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants")
os.makedirs(out, exist_ok=True)
for v in VARIANTS:
    tag = "_".join("%s%s" % (k.replace("FDL_", ""), x) for k, x in v.items())
    name = os.path.join(out, "libfiedler_%s.so" % tag)
    b.build(defines=tuple("%s=%s" % (k, x) for k, x in v.items()), out=name)
    print(name)
