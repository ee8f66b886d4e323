"""Level text codec (amaze/level.py:83-145) vs the reference's own outputs (codec.npz):
encode is byte-identical, decode round-trips, malformed texts raise LevelParseError with
the reference's message, line and column."""

import numpy as np
import pytest

from oracle import amaze_np as onp

from .helpers import rows_to_records


def _levels(z):
    import paper_2311_12716_b200 as amz

    p = onp.Params(height=13, width=13)
    out = []
    for walls, agent, adir, goal in onp.unpack_levels(rows_to_records(z["codec_levels"]), p):
        out.append(amz.MazeLevel(walls, agent, adir, goal))
    return out


def test_encode_matches_reference(golden):
    import paper_2311_12716_b200 as amz

    z = golden("codec")
    for lv, text in zip(_levels(z), z["codec_texts"]):
        assert amz.encode_level(lv) == str(text)


def test_decode_round_trip(golden):
    import paper_2311_12716_b200 as amz

    z = golden("codec")
    for lv, text in zip(_levels(z), z["codec_texts"]):
        assert amz.decode_level(str(text), expected_shape=(13, 13)).key() == lv.key()


def test_decode_errors_match_reference(golden):
    import paper_2311_12716_b200 as amz

    z = golden("codec")
    for t, msg, line, col in zip(z["codec_bad"], z["codec_bad_msg"], z["codec_bad_line"], z["codec_bad_col"]):
        t = str(t)
        shape = (3, 5) if t.startswith("######") else None
        if str(msg) == "ok":
            amz.decode_level(t, expected_shape=shape)
            continue
        with pytest.raises(amz.LevelParseError) as e:
            amz.decode_level(t, expected_shape=shape)
        assert (str(e.value), e.value.line, e.value.col) == (str(msg), int(line), int(col))
