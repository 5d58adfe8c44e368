"""Build an experimental libme.so variant (extra -D flags) for A/B timing on the GPU:
    python tools/build_variant.py NAME -DFLAG[=V] ...  -> paper_0806_0689_b200/variants/libme_NAME.so
Select it at run time with ME_LIBRARY=<path> (paper_0806_0689_b200/me.py).  Variants are
git-ignored build artefacts; the product is libme.so."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0806_0689_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(b.HERE, "variants")
os.makedirs(out, exist_ok=True)
so = os.path.join(out, f"libme_{name}.so")
import subprocess  # noqa: E402
cmd = [b.NVCC, *b.NVCC_FLAGS, *flags, "-o", so, os.path.join(b.CSRC, "me_api.cu")]
print(" ".join(cmd))
subprocess.check_call(cmd)
print(so)
