"""Policy-in-the-loop rollout throughput: eager per-step launches vs
one CUDA-graph replay per step.  The policy is a maze student net of the reference's
architecture (agents/models.py: tile/dir embeddings -> Linear(., 128) -> GRUCell(., 256)
-> policy/value heads), random init, float32, torch on the GPU."""
import sys
import time

import torch
from torch import nn

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402


class StudentNet(nn.Module):
    def __init__(self, view=5, n_actions=3, tile_dim=8, dir_dim=4, enc=128, hid=256):
        super().__init__()
        self.tile_embed = nn.Embedding(4, tile_dim)
        self.dir_embed = nn.Embedding(4, dir_dim)
        self.encoder = nn.Linear(view * view * tile_dim + dir_dim, enc)
        self.cell = nn.GRUCell(enc, hid)
        self.policy_head = nn.Linear(hid, n_actions)
        self.value_head = nn.Linear(hid, 1)
        self.hid = hid

    def initial_hidden(self, n):
        return torch.zeros(n, self.hid, device=self.policy_head.weight.device)

    def forward(self, obs, hidden):
        x = torch.cat([self.tile_embed(obs["view"]).flatten(1), self.dir_embed(obs["dir"])], dim=-1)
        h = self.cell(torch.relu(self.encoder(x)), hidden)
        return self.policy_head(h), self.value_head(h).squeeze(-1), h


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    torch.manual_seed(0)
    net = StudentNet().cuda().eval()
    actor = amz.TorchPolicyActor(net)
    P = amz.StaticParams()
    out = {}
    for name in ("eager", "graph"):
        env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
        start = env.reset(amz.RngStream.from_seed(1), P)
        gr = amz.GraphRollout(actor, env, T) if name == "graph" else None
        run = (lambda r, s: gr(r, s, copy=False)) if gr else (lambda r, s: amz.rollout(r, actor, env, s, T, P))
        traj, cur = run(amz.RngStream.from_seed(2), start)  # warm-up (and capture)
        torch.cuda.synchronize()
        ts = []
        for i in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record()
            traj, cur = run(amz.RngStream.from_seed(3 + i), cur)
            b.record()
            torch.cuda.synchronize()
            ts.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
        ms = sorted(x[0] for x in ts)[1]
        out[name] = ms
        print(f"{name}: B={B} T={T} {ms:.2f} ms/rollout, {B * T / (ms * 1e-3):.3e} lane-steps/s (wall {sorted(x[1] for x in ts)[1]:.2f} ms)")
    print(f"graph speed-up x{out['eager'] / out['graph']:.2f}")


if __name__ == "__main__":
    main()
