"""Link a variant of libpfb200.so with extra nvcc flags for one source (A/B experiments).

usage: python tools/build_variant.py NAME SOURCE.cu [-DFLAG ...]   ->  ab/NAME.so
"""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_15217_b200 import build as B

name, src, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out = Path("ab"); out.mkdir(exist_ok=True)
obj = Path(f"/tmp/variant_{name}.o")
srcp = B.CSRC / src
subprocess.run([B.NVCC, *B.NVCC_FLAGS, *extra, "-c", str(srcp), "-o", str(obj)], check=True, capture_output=True)
objs = [str(obj) if o.name == srcp.name + ".o" else str(o) for o in sorted(B.OBJDIR.glob("*.o"))]
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out / f"{name}.so"), *objs, "-lstdc++"], check=True)
print(out / f"{name}.so")
