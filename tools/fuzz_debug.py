"""Re-run a fuzz configuration with options toggled (diagnostics)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from tests.test_gpu_fuzz import _config
    from tests.test_gpu_parity import _check, _make, _run

    dev = torch.device("cuda", 0)
    for seed in map(int, sys.argv[1:]):
        B, Hq, Hkv, N, k, W, pin, combine, n_ctx, opts = _config(seed)
        for name, over in [("as-is", {}), ("parts0", {"parts": 0}), ("pin0", {}), ("win0", {}),
                           ("parts0+list", {"parts": 0, "list_gather": True})]:
            o = dict(opts, **over)
            p = 0 if name == "pin0" else pin
            w = 0 if name == "win0" else W
            rng = np.random.default_rng(10_000 + seed)
            q, K, V = _make(rng, B, Hq, Hkv, N + W + 4)
            out, idx, sc = _run(q, K, V, n_ctx, k, dev, n_win=[w] * B, pinned_prefix=p, combine=combine, **o)
            torch.cuda.synchronize()
            try:
                _check(q, K, V, n_ctx, k, out, idx, sc, n_win=[w] * B, combine=combine, pinned=p)
                print(seed, name, "ok")
            except AssertionError as e:
                print(seed, name, "FAIL", str(e).splitlines()[0][:80])


if __name__ == "__main__":
    main()
