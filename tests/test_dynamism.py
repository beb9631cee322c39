"""Budget-dynamism summaries (collect_dynamism, pipeline.py:420-462) against
the reference's own output on the same tagged budgets (tests/golden/dynamism.npz,
written by oracle/gen_golden.py), and the run-CSV layout (reporting.py:35-60).
CPU only."""

import os

import numpy as np
import pytest

from paper_2502_02770_b200 import dynamism as dy

GOLD = os.path.join(os.path.dirname(__file__), "golden", "dynamism.npz")


class _R:
    def __init__(self, b1):
        self.b1 = b1


def test_collect_dynamism_matches_reference():
    g = np.load(GOLD)
    reps = [dy.TaggedReport(*map(int, t), report=_R(int(b))) for t, b in zip(g["tags"], g["b1"])]
    st = dy.collect_dynamism(reps, bins=12)
    np.testing.assert_allclose([st.overall_mean, st.overall_std], g["overall"], rtol=1e-12)
    for axis in dy.AXES:
        a = st.axes[axis]
        np.testing.assert_allclose([a.mean, a.std, a.min, a.max], g[f"{axis}/summary"], rtol=1e-12)
        np.testing.assert_allclose(np.array(sorted(a.group_means.items()), dtype=np.float64), g[f"{axis}/groups"])
        np.testing.assert_allclose(a.histogram_edges, g[f"{axis}/edges"])
        assert list(a.histogram_counts) == g[f"{axis}/counts"].tolist()


def test_collect_dynamism_rejects_bad_input():
    with pytest.raises(ValueError):
        dy.collect_dynamism([])
    r = dy.TaggedReport(0, 0, 0, 0, _R(3))
    with pytest.raises(ValueError):
        dy.collect_dynamism([r, r])


def test_run_csv_layout(tmp_path):
    assert dy.format_value(True) == "1" and dy.format_value(0.1 + 0.2) == "0.3" and dy.format_value(7) == "7"
    p = tmp_path / "run.csv"
    dy.write_run_csv(p, [[0, 1, 2, 3, 0, False] + [1.0] * 18])
    lines = p.read_text().splitlines()
    assert lines[0].split(",") == dy.RUN_COLUMNS and lines[1].startswith("0,1,2,3,0,0,1,")
