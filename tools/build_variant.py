"""Build the library with extra nvcc defines into another path (A/B runs:
VP_LIB=<path> python bench.py ...). usage: build_variant.py OUT.so -DNAME=V ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
cmd = ["nvcc", *ge.NVCC_FLAGS, *defs, "-I", os.path.join(ge.ROOT, "include"), "-o", out, *ge._sources()]
subprocess.run(cmd, check=True, cwd=ge.ROOT)
print(out)
