"""Development aid: link a variant of libdrk_b200.so with some translation units
recompiled with extra nvcc flags.  usage:
  python scripts/build_variant.py OUT.so 'drk_raster_bwd.cu:-DDRK_BWDF_MINB=2' ...
Run it with DRK_LIB_PATH=OUT.so (the product lib stays untouched)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_11752_b200 import build as b

out = sys.argv[1]
spec = dict(a.split(":", 1) for a in sys.argv[2:])
b.build()
objs = []
for src, fmad in b.SOURCES.items():
    o = os.path.join(b.OBJ, src.replace(".cu", ".o"))
    if src in spec:
        vo = out + "." + src.replace(".cu", ".o")
        cmd = [b.NVCC, *b.COMMON, f"--fmad={'true' if fmad else 'false'}", *spec[src].split(), "-c",
               os.path.join(b.CSRC, src), "-o", vo]
        subprocess.run(cmd, check=True)
        o = vo
    objs.append(o)
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", out, *objs, "-lcudart", "-ldl"], check=True)
print(out)
