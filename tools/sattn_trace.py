"""Pipeline timeline of the sparse attention kernel's CTA 0 (dev tool; needs a library built with
-DMISA_SATTN_TRACE):  python tools/variant_lib.py /tmp/sattn_tr.so -DMISA_SATTN_TRACE
                      python tools/sattn_trace.py /tmp/sattn_tr.so"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_07363_b200 import _lib
lib = _lib.load(sys.argv[1])
from paper_2605_07363_b200.sparse_attention import sparse_attention

T, L, H, d, k = 148 * 40, 131072, 128, 128, 2048
g = torch.Generator(device="cuda").manual_seed(0)
kv = torch.randn(L, d, device="cuda", generator=g).bfloat16()
q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
topk = torch.sort(torch.randint(0, L, (T, k), device="cuda", generator=g), 1).values.int()
for _ in range(2):
    sparse_attention(q, kv, topk, d)
torch.cuda.synchronize()
buf = np.zeros((16, 1024), np.int64)
raw = ctypes.CDLL(sys.argv[1])
assert raw.misa_sattn_trace_copy(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["p_empty", "p_issued", "qk_go", "pfull_seen", "s_tfull", "s_max", "s_P", "s_pempty", "s_pfull",
         "q_tma", "q_full", "s_ofull", "s_epi_done", "oempty"]
t0 = buf[2][0]
for gg in range(64, 80):
    print(gg, " ".join(f"{names[e]}={buf[e][gg] - t0:>9d}" for e in (0, 1, 2, 4, 5, 6, 7, 8, 3)))
dd = lambda e0, e1, r: np.median(buf[e1][r] - buf[e0][r])
r = slice(40, 600)
print("median per tile: tfull->max", dd(4, 5, r), "max->P", dd(5, 6, r), "P->pempty", dd(6, 7, r),
      "pempty->pfull", dd(7, 8, r), "pfull_arrive->seen", dd(8, 3, r))
print("period (s_tfull diff)", np.median(np.diff(buf[4][40:600])), "qk_go->tfull", dd(2, 4, r))
print("rows: q_tma", np.diff(buf[9][:12]), "\n qfull-q_tma", (buf[10] - buf[9])[:12], "\n epi", (buf[12] - buf[11])[:12])
# one row boundary, every event in time order
rowstart = np.cumsum([0] + [16] * 64)  # every row of this workload has k = 2048 tokens = 16 tiles
ev = []
for r in (4, 5):
    for e, nm in ((9, "q_tma"), (10, "q_full"), (11, "s_ofull"), (12, "s_epi_done"), (13, "oempty")):
        ev.append((buf[e][r], f"{nm}[row {r}]"))
for gg in range(rowstart[4] + 13, rowstart[5] + 3):
    for e in (0, 1, 2, 4, 5, 6, 7, 8, 3):
        ev.append((buf[e][gg], f"{names[e]}[{gg}]"))
for tt, nm in sorted(ev):
    print(f"{tt - t0:>9d} {nm}")
