"""Build a variant of libdvla_b200.so with extra -D flags on one source into
tools/_variants/<name>.so (experiments; select with DVLA_B200_LIB=...).

    python tools/build_variant.py NAME token_loss.cu -DDVLA_FUSED_W=10 -DDVLA_FUSED_CTAS=2
"""
import os, subprocess, sys
from pathlib import Path
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13276_b200 import build as B

name, src, *defs = sys.argv[1:]
src_path = Path(src) if "/" in src else B.CSRC / src   # a modified copy replaces its namesake
src = src_path.name
B.build()
out = B.ROOT / "tools" / "_variants"
out.mkdir(exist_ok=True)
obj = out / f"{name}.{src}.o"
r = subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(src_path), "-o", str(obj)],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
objs = [o for o in B.OBJDIR.glob("*.o") if o.name != src + ".o"] + [obj]
r = subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out / f"{name}.so"),
                    *map(str, objs), "-ldl"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(r.stderr[-2000:] if r.stderr else "", out / f"{name}.so")
