"""Build an experimental variant of the library with extra -D flags:
python tools/build_variant.py NAME -DRUN_U=8 ..."""
import os, subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_06348_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = B.HERE / f"libalto_b200_{name}.so"
bdir = B.BUILD.parent / f"variant_{name}"
bdir.mkdir(parents=True, exist_ok=True)
objs = []
procs = []
for src in B._sources():
    obj = bdir / (src.stem + ".o")
    objs.append(obj)
    procs.append(subprocess.Popen([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", str(src), "-o", str(obj)],
                                  stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL))
assert all(p.wait() == 0 for p in procs)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart", "-ldl"], check=True)
print(out)
