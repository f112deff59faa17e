"""Phase trace of the v5 selector: builds csrc/*.cu with -DMISA_SEL_TRACE into /tmp, runs a
MISA layer, prints median cycles per phase for CTA 0's first rows.  (Dev tool, not product.)"""
import ctypes, os, subprocess, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2605_07363_b200 import _build
out = "/tmp/libmisa_trace.so"
objs = []
for src in _build.SOURCES:
    o = f"/tmp/trace_{src}.o"
    subprocess.check_call([_build._nvcc(), *_build.ARCH, *_build.FLAGS, "-DMISA_SEL_TRACE", "-c",
                           os.path.join(_build.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([_build._nvcc(), *_build.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs, "-cudart", "static"])
from paper_2605_07363_b200 import _lib
_lib.load(out)  # first load wins: the engine below uses the traced build
import torch
from paper_2605_07363_b200 import IndexerEngine, prepare_inputs
L = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "-" else 131072
g = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
Q = torch.randn(L, 64, 128, device="cuda", generator=g).bfloat16()
W = torch.softmax(torch.randn(L, 64, device="cuda", generator=g), -1).float()
x = prepare_inputs(K, Q, W)
eng = IndexerEngine(os.environ.get("METHOD", "misa"), beta=float(os.environ["BETA"]) if "BETA" in os.environ else None)
eng.run_prepared(x); eng.run_prepared(x)
torch.cuda.synchronize()
lib = _lib.load()
lib.misa_debug_sel_trace.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * (64 * 16))()
lib.misa_debug_sel_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 16).astype(np.int64)
names = (sys.argv[2] if len(sys.argv) > 2 else "top,meta,hist,level,collect,rank,pass3,scan,out").split(",")

d = np.diff(a[:, :9], axis=1)
ok = (a[:, 8] > 0)
print("rows", ok.sum(), "median cycles per phase:")
for i, nm in enumerate(names[1:]):
    print(f"  {names[i]:>9s}->{nm:<9s} {int(np.median(d[ok, i])):8d}")
if (a[ok, 14] > 0).any():
    print("  issue only", int(np.median(a[ok, 14] - a[ok, 5])), " load_meta", int(np.median(a[ok, 6] - a[ok, 14])))
print("  row total", int(np.median(a[ok, 8] - a[ok, 0])), " row-to-row", int(np.median(np.diff(a[ok, 0]))))
cut = a[:, 9:14]
okc = ok & (cut[:, 0] > 0) & (cut[:, 4] > 0)
if okc.any():
    seq = np.concatenate([a[:, 2:3], cut], 1)  # extract end -> cut marks
    dd = np.diff(seq, axis=1)
    for i, nm in enumerate(["minmax", "hist", "scan+lvl", "collect", "rank"]):
        print(f"  cut:{nm:<9s} {int(np.median(dd[okc, i])):8d}")
    print("  boundary bin sizes:", a[okc, 15][:20].tolist())
