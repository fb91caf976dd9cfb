"""Build libtlru.so with extra -D tunables into paper_2510_15152_b200/variants/libtlru_<name>.so
(measurement A/B only; loaded when TLRU_LIB_VARIANT=<name>):
    python tools/build_variant.py NAME -DTLRU_WIN_G=8 [...]"""
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(G.PKG, "variants")
os.makedirs(out_dir, exist_ok=True)
srcs = sorted(os.path.join(G.CSRC, f) for f in os.listdir(G.CSRC) if f.endswith(".cu"))
cflags = [f for f in G.NVCC_FLAGS if f != "-shared"] + defs
with tempfile.TemporaryDirectory() as td:
    objs = [os.path.join(td, os.path.basename(s) + ".o") for s in srcs]
    cmds = [[G._nvcc(), *cflags, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o] for s, o in zip(srcs, objs)]
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for f in [ex.submit(subprocess.check_call, c, cwd=ROOT) for c in cmds]:
            f.result()
    subprocess.check_call([G._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                           os.path.join(out_dir, f"libtlru_{name}.so"), *objs], cwd=ROOT)
print("built", name)
