"""Golden per-layer budgets from the LIVE reference (budget.py), for tests/test_budget.py.

Run in the development container (the reference tree does not exist on the GPU box):

    python tests/golden/make_budget_golden.py

Writes tests/golden/budget_cases.json: for each case the strategy, its arguments and either
the reference's k_per_layer or the name of the exception it raised.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "budget_cases.json"


def main() -> None:
    import numpy as np

    sys.path.insert(0, str(REF))
    from topk_kv import budget as B  # noqa: E402

    rng = np.random.default_rng(2502)
    cases = []

    def run(kind, args, fn):
        try:
            ks = list(fn().k_per_layer)
            cases.append({"kind": kind, "args": args, "k": ks})
        except Exception as exc:  # noqa: BLE001 — the exception class is the expected outcome
            cases.append({"kind": kind, "args": args, "error": type(exc).__name__})

    for L, T in [(1, 1), (4, 4), (4, 3), (32, 32), (32, 31), (32, 8192), (32, 524288), (7, 100), (12, 13)]:
        run("uniform", [L, T], lambda L=L, T=T: B.uniform_budget(L, T))
        run("linear", [L, T], lambda L=L, T=T: B.linear_budget(L, T))
    for _ in range(40):
        L = int(rng.integers(1, 40))
        T = int(rng.integers(max(1, L - 2), 50000))
        run("linear", [L, T], lambda L=L, T=T: B.linear_budget(L, T))
        ent = [float(x) for x in np.round(rng.gamma(1.5, 2.0, size=L), 6)]
        if rng.random() < 0.3:
            ent[int(rng.integers(0, L))] = 0.0
        run("entropy", [L, T, ent], lambda L=L, T=T, ent=ent: B.entropy_budget(L, T, ent))
    # heavy skew: zero-share layers lifted to 1
    run("entropy", [6, 8, [0.0, 0.0, 0.0, 100.0, 0.0, 0.0]],
        lambda: B.entropy_budget(6, 8, [0.0, 0.0, 0.0, 100.0, 0.0, 0.0]))
    run("entropy", [5, 5, [1.0, 2.0, 3.0, 4.0, 5.0]], lambda: B.entropy_budget(5, 5, [1.0, 2.0, 3.0, 4.0, 5.0]))
    run("entropy", [3, 10, [1.0, -1.0, 1.0]], lambda: B.entropy_budget(3, 10, [1.0, -1.0, 1.0]))
    run("entropy", [3, 10, [1.0, 1.0]], lambda: B.entropy_budget(3, 10, [1.0, 1.0]))
    for spec, L in [("uniform:256", 32), ("linear:8192", 32), ("explicit:[1,2,3]", 3), ("explicit:[1,2]", 3),
                    ("bogus:1", 4), ("linear:abc", 4), ("entropy:100", 4), ("uniform:0", 4)]:
        run("spec", [spec, L], lambda spec=spec, L=L: B.parse_budget_spec(spec, L))
    run("layer_budget", [[3, 4, 5], 12], lambda: B.LayerBudget((3, 4, 5), 12))
    run("layer_budget", [[3, 4, 5], 13], lambda: B.LayerBudget((3, 4, 5), 13))
    run("layer_budget", [[3, 0, 5], 0], lambda: B.LayerBudget((3, 0, 5)))
    OUT.write_text(json.dumps({"source": "reference budget.py (live)", "cases": cases}, indent=0) + "\n")
    print(f"{len(cases)} cases -> {OUT}")


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_golden"))
    main()
