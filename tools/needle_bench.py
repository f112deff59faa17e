"""Needle retrieval at full length (C4: L = 131072 keys): structured data for the recall-vs-DSA
numbers SURVEY.md §8(d) asks for beside the random-data IoU.

R query rows share one key sequence; row r's 32-key needle (``gen_needle_workload``'s
construction, ``workload.py:143-199``: margin * unit(q_target) + noise, target = the row's
top-gate head) sits at depth r / (R - 1).  Every row sees the whole prefix.  Reported per
method: needle recall (fraction of needle keys in the row's top-k) and the top-k set
recall against DSA's top-k on the same rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_07363_b200 import IndexerEngine  # noqa: E402


def needle_inputs(L=131072, R=16, H=64, d=128, needle_len=32, margin=10.0, noise=0.01, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.randn(L, d, device="cuda", generator=g)
    Q = torch.randn(R, H, d, device="cuda", generator=g)
    W = torch.softmax(torch.randn(R, H, device="cuda", generator=g), -1)
    spans = []
    for r in range(R):
        tgt = int(W[r].argmax())
        start = int((r / max(R - 1, 1)) * (L - needle_len))
        u = Q[r, tgt] / Q[r, tgt].norm()
        K[start:start + needle_len] = margin * u + noise * torch.randn(needle_len, d, device="cuda", generator=g)
        spans.append((start, start + needle_len))
    return K.bfloat16(), Q.bfloat16(), W.float(), spans


def needle_numbers(L=131072, R=16, k=2048, h=8, B=1024, kprime=8192):
    K, Q, W, spans = needle_inputs(L, R)
    prefix = torch.full((R,), L, dtype=torch.int32, device="cuda")
    sel = {}
    for m in ("dsa", "misa", "misa_hier"):
        eng = IndexerEngine(m, budget_k=k, active_heads_h=h, block_size=B, candidate_kprime=kprime)
        sel[m] = eng.run(K, Q, W, prefix).topk.cpu()
    out = {"what": f"{R} rows x L={L} keys, 32-key margin-10 needle per row at depth r/{R - 1} "
                   "aligned with the row's top-gate head; recall of the needle and of DSA's top-k set",
           "needle_recall": {}, "topk_recall_vs_dsa": {}}
    for m, t in sel.items():
        hit = sum(len(set(t[r].tolist()) & set(range(*spans[r]))) for r in range(R))
        out["needle_recall"][m] = round(hit / (32 * R), 4)
        if m != "dsa":
            same = sum(len(set(t[r].tolist()) & set(sel["dsa"][r].tolist())) for r in range(R))
            out["topk_recall_vs_dsa"][m] = round(same / (k * R), 4)
    return out


if __name__ == "__main__":
    import json
    print(json.dumps(needle_numbers()))
