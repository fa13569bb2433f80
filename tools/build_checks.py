"""Link ab/checks.so: every source built with -DPF_CHECKS (device-side bounds traps, see
csrc/pf_common.cuh).  Run the GPU tests against it with PF_B200_LIB=$PWD/ab/checks.so."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2404_15217_b200 import build as B  # noqa: E402

out = Path(__file__).resolve().parents[1] / "ab"
out.mkdir(exist_ok=True)
objs = []
for src in B._sources():
    obj = Path(f"/tmp/checks_{src.name}.o")
    if src.suffix == ".cu":
        cmd = [B.NVCC, *B.NVCC_FLAGS, "-DPF_CHECKS", "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *B.CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    subprocess.run(cmd, check=True, capture_output=True)
    objs.append(str(obj))
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out / "checks.so"), *objs, "-lstdc++"], check=True)
print(out / "checks.so")
