"""Build variant libraries for same-box A/B timing: python tools/ab_build.py NAME -DFOO=1 [-D...]
-> abtest/NAME.so (git-ignored, travels to the GPU box); run with RALPB_LIB=abtest/NAME.so."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1901_05803_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
objdir = ROOT / "abtest" / f"{name}_obj"
objdir.mkdir(parents=True, exist_ok=True)
procs = []
for src in b.sources():
    obj = objdir / (src.stem + ".o")
    procs.append(subprocess.Popen([b.NVCC, *b.ARCH, *b.FLAGS, *defs, "-c", str(src), "-o", str(obj)]))
assert all(p.wait() == 0 for p in procs), "nvcc failed"
out = ROOT / "abtest" / f"{name}.so"
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(out), *map(str, sorted(objdir.glob("*.o"))), "-lcudart_static",
                "-ldl", "-lrt", "-lpthread"], check=True)
print(out)
