"""Curriculum metrics kernel (k_level_metrics) vs the reference's env_metrics fixtures
(amaze/metrics.py:21-31, BFS of amaze/pathfinding.py:116-135) and the numpy oracle."""

import numpy as np
import pytest

from oracle import amaze_np as onp

from .helpers import rows_to_records

pytestmark = pytest.mark.gpu


def _dev_levels(rows):
    import torch

    rec = rows_to_records(rows)
    return torch.from_numpy(rec.view(np.int32).reshape(len(rows), 8).copy()).cuda()


@pytest.mark.parametrize("name", ["default", "dense", "small9", "wide", "assets"])
def test_level_metrics_match_reference(golden, name):
    import paper_2311_12716_b200 as amz

    z = golden("metrics")
    H, W = (int(x) for x in z[f"m_{name}_meta"])
    P = amz.StaticParams(height=H, width=W, wall_budget=min(60, (H - 2) * (W - 2) - 2))
    m = amz.level_metrics(_dev_levels(z[f"m_{name}_levels"]), P)
    assert np.array_equal(m["n_walls"].cpu().numpy(), z[f"m_{name}_nwalls"])
    assert np.array_equal(m["shortest_path_length"].cpu().numpy(), z[f"m_{name}_spl"])
    assert np.array_equal(m["solvable"].cpu().numpy(), z[f"m_{name}_solvable"])
    assert np.array_equal(m["passable_ratio"].cpu().numpy(), z[f"m_{name}_passable"])  # bit-exact float64


@pytest.mark.parametrize("hw,budget", [((13, 13), 60), ((12, 12), 90), ((11, 14), 100), ((5, 7), 8), ((12, 9), 50)])
def test_level_metrics_random_levels_vs_oracle(hw, budget):
    import paper_2311_12716_b200 as amz

    H, W = hw
    P = amz.StaticParams(height=H, width=W, wall_budget=min(budget, (H - 2) * (W - 2) - 2))
    lv = amz.sample_levels(amz.RngStream(11, (5,)), 3000, P)
    m = amz.level_metrics(lv, P)
    host = amz.amaze.to_host_levels(lv, P)
    p = onp.Params(height=H, width=W)
    want = np.array([onp.env_metrics((np.asarray(x.walls), tuple(x.agent_pos), x.agent_dir, tuple(x.goal_pos)))
                     for x in host], dtype=object)
    assert np.array_equal(m["n_walls"].cpu().numpy(), want[:, 0].astype(np.int64))
    assert np.array_equal(m["shortest_path_length"].cpu().numpy(), want[:, 1].astype(np.int64))
    assert np.array_equal(m["solvable"].cpu().numpy(), want[:, 2].astype(bool))
    assert np.array_equal(m["passable_ratio"].cpu().numpy(), want[:, 3].astype(np.float64))
    del p


def test_env_metrics_single_level_api():
    import paper_2311_12716_b200 as amz

    P = amz.StaticParams()
    lv = amz.sample_random_level(amz.RngStream(3, (1,)), P)
    em = amz.env_metrics(lv)
    w = np.asarray(lv.walls)
    want = onp.env_metrics((w, tuple(lv.agent_pos), lv.agent_dir, tuple(lv.goal_pos)))
    assert (em.n_walls, em.shortest_path_length, em.solvable, em.passable_ratio) == want
    assert amz.level_metrics(amz.sample_levels(amz.RngStream(3, (1,)), 0, P), P)["n_walls"].numel() == 0
