"""Maze levels on the host and as packed device records.

``MazeLevel`` is the host value type of the reference (``amaze/level.py:33-80``):
walls bool[H, W], agent (r, c), heading 0..3 (N, E, S, W), goal (r, c).  On the GPU a
level is one 32-byte ``amz_level_t`` record (include/amaze_b200.h): the interior wall
bits (cell (r, c) -> bit (r-1)*(W-2) + (c-1)) plus the pose bytes.  A batch of levels
is a ``torch.int32`` tensor of shape [N, 8] (``LevelBatch``); conversion to/from
``MazeLevel`` lists is host-side API plumbing, not part of the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import LevelError, LevelParseError

# agent heading glyphs, amaze/level.py:29-30
AGENT_CHARS = {0: "^", 1: ">", 2: "v", 3: "<"}
CHAR_DIRS = {v: k for k, v in AGENT_CHARS.items()}

RECORD = np.dtype([("walls", "<u4", (4,)), ("agent_r", "u1"), ("agent_c", "u1"), ("agent_dir", "u1"),
                   ("goal_r", "u1"), ("goal_c", "u1"), ("pad", "u1", (3,)), ("pad2", "<u4", (2,))])
DIR_VECTORS = np.array([(-1, 0), (0, 1), (1, 0), (0, -1)], dtype=np.int64)


@dataclass
class MazeLevel:
    walls: np.ndarray  # bool [H, W]
    agent_pos: tuple
    agent_dir: int
    goal_pos: tuple

    @property
    def height(self) -> int:
        return self.walls.shape[0]

    @property
    def width(self) -> int:
        return self.walls.shape[1]

    def validate(self) -> "MazeLevel":
        """The invariants of amaze/level.py:50-66."""
        h, w = self.walls.shape
        if h < 3 or w < 3:
            raise LevelError(f"level must be at least 3x3, got {h}x{w}")
        rim = np.concatenate([self.walls[0], self.walls[-1], self.walls[:, 0], self.walls[:, -1]])
        if not rim.all():
            raise LevelError("border cells must all be walls")
        for who, (r, c) in (("agent", self.agent_pos), ("goal", self.goal_pos)):
            if not (0 < r < h - 1 and 0 < c < w - 1):
                raise LevelError(f"{who} position {(r, c)} is not an interior cell")
            if self.walls[r, c]:
                raise LevelError(f"{who} position {(r, c)} is a wall cell")
        if tuple(self.agent_pos) == tuple(self.goal_pos):
            raise LevelError(f"agent and goal share cell {tuple(self.agent_pos)}")
        if self.agent_dir not in (0, 1, 2, 3):
            raise LevelError(f"agent_dir must be in 0..3, got {self.agent_dir}")
        return self

    def key(self) -> bytes:
        """Identity: packed wall bits + int64 pose (same bytes as amaze/level.py:68-71)."""
        pose = np.array([*self.agent_pos, self.agent_dir, *self.goal_pos], dtype=np.int64)
        return np.packbits(self.walls).tobytes() + pose.tobytes()

    def copy(self) -> "MazeLevel":
        return MazeLevel(self.walls.copy(), tuple(self.agent_pos), int(self.agent_dir), tuple(self.goal_pos))

    def n_interior_walls(self) -> int:
        return int(self.walls[1:-1, 1:-1].sum())

    def __eq__(self, other) -> bool:
        return hasattr(other, "walls") and self.key() == MazeLevel.from_any(other).key()

    @staticmethod
    def from_any(lv) -> "MazeLevel":
        if isinstance(lv, MazeLevel):
            return lv
        return MazeLevel(np.asarray(lv.walls, dtype=bool), tuple(int(x) for x in lv.agent_pos), int(lv.agent_dir),
                         tuple(int(x) for x in lv.goal_pos))


def pack_levels(levels, height: int, width: int) -> np.ndarray:
    """MazeLevel-like objects -> amz_level_t records (numpy structured array)."""
    n = len(levels)
    out = np.zeros(n, dtype=RECORD)
    if n == 0:
        return out
    inner = np.stack([np.asarray(lv.walls, dtype=bool)[1:-1, 1:-1].reshape(-1) for lv in levels])
    if inner.shape[1] != (height - 2) * (width - 2):
        raise LevelError(f"levels are not {height}x{width}")
    bits = np.zeros((n, 128), dtype=np.uint8)
    bits[:, : inner.shape[1]] = inner
    words = np.packbits(bits.reshape(n, 16, 8)[:, :, ::-1], axis=-1).reshape(n, 16)
    out["walls"] = words.view("<u4").reshape(n, 4)
    out["agent_r"] = [lv.agent_pos[0] for lv in levels]
    out["agent_c"] = [lv.agent_pos[1] for lv in levels]
    out["agent_dir"] = [lv.agent_dir for lv in levels]
    out["goal_r"] = [lv.goal_pos[0] for lv in levels]
    out["goal_c"] = [lv.goal_pos[1] for lv in levels]
    return out


def unpack_levels(rec: np.ndarray, height: int, width: int) -> list:
    """amz_level_t records -> MazeLevel list."""
    rec = np.asarray(rec).view(RECORD).reshape(-1)
    n = rec.shape[0]
    ni = (height - 2) * (width - 2)
    raw = np.ascontiguousarray(rec["walls"]).view(np.uint8).reshape(n, 16, 1)
    bits = np.unpackbits(raw, axis=-1)[:, :, ::-1].reshape(n, 128)[:, :ni].astype(bool)
    out = []
    for i in range(n):
        walls = np.ones((height, width), dtype=bool)
        walls[1:-1, 1:-1] = bits[i].reshape(height - 2, width - 2)
        r = rec[i]
        out.append(MazeLevel(walls, (int(r["agent_r"]), int(r["agent_c"])), int(r["agent_dir"]),
                             (int(r["goal_r"]), int(r["goal_c"]))))
    return out


def records_to_tensor(rec: np.ndarray, device="cuda"):
    import torch

    arr = np.ascontiguousarray(rec).view(np.int32).reshape(-1, 8)
    return torch.from_numpy(arr.copy()).to(device)


def tensor_to_records(t) -> np.ndarray:
    arr = t.detach().to("cpu").contiguous().numpy().astype(np.int32, copy=False)
    return arr.reshape(-1).view(RECORD)


def encode_level(level) -> str:
    """Grid text of a level (amaze/level.py:83-97): '#' wall, '.' floor, 'G' goal,
    '^>v<' the agent by heading; one line per row, trailing newline."""
    lv = MazeLevel.from_any(level)
    walls = np.asarray(lv.walls, dtype=bool)
    h, w = walls.shape
    grid = np.where(walls, "#", ".").astype("<U1")
    grid[tuple(lv.goal_pos)] = "G"
    grid[tuple(lv.agent_pos)] = AGENT_CHARS[int(lv.agent_dir)]
    return "\n".join("".join(row) for row in grid) + "\n"


def decode_level(text: str, expected_shape: tuple | None = None) -> MazeLevel:
    """Parse grid text (amaze/level.py:100-145): blank lines skipped, ragged rows,
    wrong shape, illegal characters, duplicate / missing agent or goal raise
    LevelParseError with the 1-based line/column the reference reports; invariant
    violations of the parsed level become LevelParseError at (1, 1)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise LevelParseError("empty level text", 1, 1)
    h, w = len(lines), len(lines[0])
    for i, ln in enumerate(lines):
        if len(ln) != w:
            raise LevelParseError(f"row has length {len(ln)}, expected {w}", i + 1, len(ln) + 1)
    if expected_shape is not None and (h, w) != tuple(expected_shape):
        raise LevelParseError(f"level is {h}x{w}, expected {expected_shape[0]}x{expected_shape[1]}", 1, 1)
    walls = np.zeros((h, w), dtype=bool)
    agent_pos = agent_dir = goal_pos = None
    for r, ln in enumerate(lines):
        for c, ch in enumerate(ln):
            if ch == "#":
                walls[r, c] = True
            elif ch == ".":
                continue
            elif ch == "G":
                if goal_pos is not None:
                    raise LevelParseError("duplicate goal", r + 1, c + 1)
                goal_pos = (r, c)
            elif ch in CHAR_DIRS:
                if agent_pos is not None:
                    raise LevelParseError("duplicate agent", r + 1, c + 1)
                agent_pos, agent_dir = (r, c), CHAR_DIRS[ch]
            else:
                raise LevelParseError(f"illegal character {ch!r}", r + 1, c + 1)
    if agent_pos is None:
        raise LevelParseError("missing agent", h, w)
    if goal_pos is None:
        raise LevelParseError("missing goal", h, w)
    try:
        return MazeLevel(walls, agent_pos, agent_dir, goal_pos).validate()
    except LevelParseError:
        raise
    except LevelError as e:
        raise LevelParseError(str(e), 1, 1) from e
