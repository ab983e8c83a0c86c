"""The paper's comparisons on the GPU engine (SURVEY.md §8f row 2,
paper_2512_18126_b200/ablation.py): run_ablation's four settings
(orchestrator.cpp:451-521) and the second-layer schedule study
(orchestrator.cpp:532-578), with device-event latencies.

The reference's own ablation tests (test_orchestrator.cpp) check structure and
normalisation, not speed-ups (its times are virtual); the same holds here: the
rows, the normalisation against all-to-all / sequential P/D, and that the
settings without early exit decode every invoked agent's full output."""
import pytest

from paper_2512_18126_b200 import ablation
from paper_2512_18126_b200.configs import C1

pytestmark = pytest.mark.gpu


def test_ablation_rows_and_normalisation():
    rows = ablation.run_ablation(dict(C1), samples=2)
    assert [r["setting"] for r in rows] == ["all-to-all", "tree", "tree+overlap", "tree+overlap+ee"]
    assert rows[0]["normalized_mean"] == pytest.approx(1.0)
    for r in rows:
        assert r["samples"] == 2 and r["mean_e2e_ms"] > 0 and r["tokens_per_s"] > 0
        assert r["p50_e2e_ms"] <= r["p95_e2e_ms"] + 1e-9
    # same tree, same agents, no early exit: overlap changes time, not work
    t_tree = rows[1]["tokens_per_s"] * rows[1]["mean_e2e_ms"]
    t_ovl = rows[2]["tokens_per_s"] * rows[2]["mean_e2e_ms"]
    assert t_tree == pytest.approx(t_ovl, rel=1e-9)


def test_second_layer_study_modes():
    rows = ablation.run_second_layer_study(dict(C1), precursors=4, out_min=16, out_max=48, samples=2)
    assert [r["mode"] for r in rows] == list(ablation.MODES)
    assert rows[0]["normalized_vs_sequential"] == pytest.approx(1.0)
    assert all(r["mean_e2e_ms"] > 0 for r in rows)
