"""build_variant.py NAME 'sed-expression' [files-glob]: build build/libppfg_NAME.so
from a copy of csrc edited by the sed expression (A/B runs). Translation units
whose text is unchanged (and no header changed) reuse the in-tree objects."""
import filecmp
import glob
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1411_3656_b200 import build as B  # noqa: E402

name, expr = sys.argv[1], sys.argv[2]
B.build()  # the in-tree objects are current
d = tempfile.mkdtemp()
src = os.path.join(d, "csrc")
shutil.copytree(B.CSRC, src)
files = sorted(glob.glob(os.path.join(src, "*.cu")) + glob.glob(os.path.join(src, "*.cuh")) +
               glob.glob(os.path.join(src, "*.cpp")) +
               glob.glob(os.path.join(src, "*.h")))
if expr.startswith("git:"):  # git:REV — the csrc sources of that revision
    rev = expr[4:]
    for f in files:
        rel = os.path.relpath(os.path.join(B.CSRC, os.path.basename(f)), ROOT)
        r = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{rel}"], capture_output=True)
        if r.returncode == 0:
            open(f, "wb").write(r.stdout)
else:
    subprocess.check_call(["sed", "-i", expr, *files])
changed = [f for f in files if not filecmp.cmp(f, os.path.join(B.CSRC, os.path.basename(f)), shallow=False)]
print("changed:", [os.path.basename(f) for f in changed])
hdr_changed = any(not f.endswith(".cu") for f in changed)
objs = []
todo = []
for cu in sorted(glob.glob(os.path.join(src, "*.cu")) + glob.glob(os.path.join(src, "*.cpp"))):
    if hdr_changed or cu in changed:
        o = os.path.join(d, os.path.splitext(os.path.basename(cu))[0] + ".o")
        todo.append((cu, o))
        objs.append(o)
    else:
        objs.append(B._obj(os.path.join(B.CSRC, os.path.basename(cu))))


def cc(job):
    cu, o = job
    subprocess.check_call(B.compile_cmd(cu, o))


with ThreadPoolExecutor(max_workers=8) as ex:
    list(ex.map(cc, todo))
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
out = os.path.join(ROOT, "build", f"libppfg_{name}.so")
subprocess.check_call([B._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs])
shutil.rmtree(d)
print(out)
