"""Re-run one fuzz configuration (tests/test_gpu_fuzz.py) and print the heads whose ids differ
from the contract, optionally overriding options: python tools/fuzz_repro.py SEED [adv] [key=val ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from tests.test_gpu_fuzz import _adversarial, _config  # noqa: E402
from tests.test_gpu_parity import _make, _run  # noqa: E402

seed = int(sys.argv[1])
adv = len(sys.argv) > 2 and sys.argv[2] == "adv"
over = dict(a.split("=") for a in sys.argv[3 if adv else 2:])
B, Hq, Hkv, N, k, W, pin, combine, n_ctx, opts = _config(500 + seed if adv else seed)
for key, v in over.items():
    if key == "pin":
        pin = int(v)
    elif key == "W":
        W = int(v)
    else:
        opts[key] = None if v == "None" else (v == "True" if v in ("True", "False") else int(v))
print("cfg", B, Hq, Hkv, N, k, W, pin, combine, n_ctx, opts)
rng = np.random.default_rng((20_000 if adv else 10_000) + seed)
q, K, V = _make(rng, B, Hq, Hkv, N + W + 4)
if adv:
    K = _adversarial(seed, q, K, n_ctx)
cuda = torch.device("cuda", 0)
out, idx, sc = _run(q, K, V, n_ctx, k, cuda, n_win=[W] * B, pinned_prefix=pin, combine=combine, **opts)
torch.cuda.synchronize()
idx = idx.cpu().numpy()
sc = sc.cpu().numpy()
nbad = 0
for b in range(B):
    kb = min(k, n_ctx[b])
    for h in range(Hq):
        tail, head = idx[b, h, kb:], idx[b, h, :kb]
        if not (tail == -1).all() or len(set(head.tolist())) != kb or head.max() >= n_ctx[b]:
            nbad += 1
            if nbad <= 2:
                print("b", b, "h", h, "kb", kb, "head", head[:12], "...", head[-6:], "max", head.max())
                print("   tail", tail[:12], "non-pad", int((tail != -1).sum()), "scores", sc[b, h, :4], sc[b, h, kb:kb + 4])
print("bad heads", nbad)
