import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2502_06766_b200 as tkv
from paper_2502_06766_b200 import ops, _lib

def layout(B, Hq, Hkv, max_ctx, k):
    BH, BK = B * Hq, B * Hkv
    off = 0
    L = {}
    def take(name, n):
        nonlocal off
        L[name] = off
        off = (off + max(n, 1) + 255) // 256 * 256
    take("ticket_g", BH * 4); take("ticket_k", BH * 4); take("flag", BH * 4); take("gflag", BK * 4)
    take("fctl", (8 + 2 * BK + 5 * BH) * 4)
    take("cnt", BH * 4); take("thr", BH * 4); take("hshift", BH * 4); take("hist", BH * 4096 * 4)
    take("maxc", BH * 8); take("bktc", BH * 4); take("outc", BH * 4); take("bkt", BH * 8192 * 8)
    take("mmax", BH * 4); take("mkth", BH * 8); take("mkb", BH * 4); take("samp", BH * 4096 * 4)
    cap = max(max_ctx, 1)
    take("cand", BH * cap * 8)
    return L, cap

dev = torch.device("cuda", 0)
K = np.zeros((5, 128), np.float32); K[:, 0] = [1, 2, 1, 2, 1]
q = np.zeros(128, np.float32); q[0] = 1
Kd = torch.from_numpy(K).to(dev, torch.bfloat16)[None, None].contiguous()
qd = torch.from_numpy(q).to(dev, torch.bfloat16)[None, None].contiguous()
L, cap = layout(1, 1, 1, 5, 3)
for fused in (False, True):
    prob = ops.make_problem(1, 1, 1, 5, 5, 3, sorted=False, fused=fused)
    ws = ops.workspace_for(prob, dev)
    idx, sc = ops.topk_search(qd, Kd, 5, 3, sorted=False, fused=fused, workspace=ws)
    torch.cuda.synchronize()
    base = ws.ptr.value - ws._buf.data_ptr()
    buf = ws._buf[base:].cpu().numpy()
    u32 = lambda name, n: buf[L[name]:L[name] + 4 * n].view(np.uint32)
    u64 = lambda name, n: buf[L[name]:L[name] + 8 * n].view(np.uint64)
    cnt = int(u32("cnt", 1)[0])
    cand = u64("cand", cap)
    print("fused", fused, "idx", idx.cpu().numpy().ravel(), "cnt", cnt, "thr", u32("thr", 1), "shift", u32("hshift", 1))
    print("  cand gids", [int((~int(c)) & 0xffffffff) for c in cand[:cnt]], "keys", [hex(int(c) >> 32) for c in cand[:cnt]])
    print("  mkth", hex(int(u64("mkth", 1)[0])), "mkb", buf[L["mkb"]:L["mkb"]+4].view(np.int32), "outc", u32("outc", 1), "fctl", u32("fctl", 8 + 2 + 5))
    h = u32("hist", 4096); nz = np.flatnonzero(h); print("  hist nz", list(zip(nz.tolist(), h[nz].tolist())))
