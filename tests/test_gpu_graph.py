"""The captured DR iteration (graph.DRIterationGraph) equals the eager calls bit for
bit: reset(root.fold_in(it)) -> rollout_actions -> gae_and_scores, for consecutive
iterations, a jump, and the host-I/O forms (with and without the overlapped copies)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T, G, L = 512, 64, 0.995, 0.98


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _eager(root, it, acts, vals, last, p):
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    res = env.reset(root.fold_in(it), p)
    tr, cur = amz.rollout_actions(env, res, acts, p)
    o = amz.gae_and_scores(tr.rewards, vals, tr.dones, last, G, L)
    return res, tr, cur, o


def _inputs(seed, vdt=torch.float64):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return (torch.randint(0, 3, (T, B), generator=g, device="cuda", dtype=torch.uint8),
            torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64).to(vdt),
            torch.rand((B,), generator=g, device="cuda", dtype=torch.float64).to(vdt))


def _same(gr, res, tr, cur, o):
    assert torch.equal(gr.out["reset_view"], res.observation["view"].reshape(B, 5, 5))
    assert torch.equal(gr.out["view"], tr.obs["view"]) and torch.equal(gr.out["dir"], tr.obs["dir"])
    assert torch.equal(gr.out["rewards"], tr.rewards) and torch.equal(gr.out["dones"], tr.dones)
    assert torch.equal(gr.out["final_view"], cur.obs["view"])
    for k in ("advantages", "returns", "scores", "max_returns"):
        assert torch.equal(gr.gae[k], o[k]), k


def test_graph_replays_equal_eager_iterations():
    p = amz.StaticParams()
    root = amz.RngStream.from_seed(42)
    acts, vals, last = _inputs(1)
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), root, T, p, G, L).capture()
    gr.inputs[0]["actions"].copy_(acts)
    gr.inputs[0]["values"].copy_(vals)
    gr.inputs[0]["last"].copy_(last)
    for it in [0, 1, 2, 7, 8]:  # in order, then a jump
        gr.step(it)
        torch.cuda.synchronize()
        _same(gr, *_eager(root, it, acts, vals, last, p))


@pytest.mark.parametrize("overlap,copy_mode,streams", [(False, "auto", 1), (True, "kernel", 1), (True, "engine", 1),
                                                       (True, "engine", 3), (True, "auto", 1)])
@pytest.mark.parametrize("vdt", [torch.float64, torch.float32])
def test_graph_host_io(overlap, copy_mode, streams, vdt):
    p = amz.StaticParams()
    root = amz.RngStream.from_seed(3)
    acts, vals, last = _inputs(2, vdt)
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), root, T, p, G, L,
                          value_dtype=vdt, host_io=True, overlap=overlap, copy_mode=copy_mode, copy_streams=streams)
    gr.host_inputs["actions"].copy_(acts.cpu())
    gr.host_inputs["values"].copy_(vals.cpu())
    gr.host_inputs["last"].copy_(last.cpu())
    gr.capture()
    if copy_mode == "auto" and overlap:
        gr.calibrate(rounds=2, steps=2)  # real steps, counter restored: iteration 0 is next
        assert gr.next_it == 0 and set(gr.calibration_ms) == {False, True}
    for it in range(4):
        gr.step()
        torch.cuda.synchronize()
        res, tr, cur, o = _eager(root, it, acts, vals, last, p)
        _same(gr, res, tr, cur, o)
        assert np.array_equal(gr.host_result[0].numpy(), o["scores"].cpu().numpy())
        assert np.array_equal(gr.host_result[1].numpy(), o["max_returns"].cpu().numpy())
