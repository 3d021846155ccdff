"""Per-layer k budgets (budget.py) against golden outcomes from the live reference
(tests/golden/budget_cases.json, made by tests/golden/make_budget_golden.py)."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2502_06766_b200 import budget as B
from paper_2502_06766_b200 import errors

CASES = json.loads((Path(__file__).parent / "golden" / "budget_cases.json").read_text())["cases"]


def _run(case):
    kind, args = case["kind"], case["args"]
    if kind == "uniform":
        return B.uniform_budget(*args)
    if kind == "linear":
        return B.linear_budget(*args)
    if kind == "entropy":
        return B.entropy_budget(*args)
    if kind == "spec":
        return B.parse_budget_spec(*args)
    if kind == "layer_budget":
        return B.LayerBudget(tuple(args[0]), args[1])
    raise AssertionError(kind)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_budget_matches_reference(i):
    case = CASES[i]
    if "error" in case:
        with pytest.raises(getattr(errors, case["error"])):
            _run(case)
    else:
        got = _run(case)
        assert list(got.k_per_layer) == case["k"]
        assert got.total == sum(case["k"]) and got.n_layers == len(case["k"])


def test_entropy_spec_reads_file(tmp_path):
    p = tmp_path / "ent.json"
    p.write_text(json.dumps([0.5, 1.0, 2.0, 0.0]))
    b = B.parse_budget_spec(f"entropy:100:{p}", 4)
    assert b.total == 100 and b.n_layers == 4 and b[2] == max(b.k_per_layer)
    with pytest.raises(errors.ConfigError):
        B.parse_budget_spec(f"entropy:100:{tmp_path / 'missing.json'}", 4)
