"""Shared test helpers (fixture decoding)."""

import numpy as np

from oracle import amaze_np as onp


def rows_to_records(rows):
    rec = np.zeros(len(rows), dtype=onp.LEVEL_DTYPE)
    rec["walls"] = rows[:, :4].astype(np.uint32)
    rec["agent_r"], rec["agent_c"], rec["agent_dir"] = rows[:, 4], rows[:, 5], rows[:, 6]
    rec["goal_r"], rec["goal_c"] = rows[:, 7], rows[:, 8]
    return rec


def records_to_rows(rec):
    return np.stack([rec["walls"][:, 0], rec["walls"][:, 1], rec["walls"][:, 2], rec["walls"][:, 3],
                     rec["agent_r"], rec["agent_c"], rec["agent_dir"], rec["goal_r"], rec["goal_c"]],
                    axis=1).astype(np.int64)


def tensor_rows(t):
    arr = t.detach().cpu().contiguous().numpy().astype(np.int32).reshape(-1).view(onp.LEVEL_DTYPE)
    return records_to_rows(arr)
