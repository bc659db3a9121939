"""Host-side chunk planning of the pipelined round trip (no GPU)."""
from paper_1303_4994_b200.pipeline import chunk_weights


def test_chunk_weights_equal_without_taper():
    assert chunk_weights(5) == [1, 1, 1, 1, 1]
    assert chunk_weights(3, taper=1) == [1, 1, 1]


def test_chunk_weights_taper_ramps_and_caps():
    assert chunk_weights(8, taper=4) == [1, 2, 4, 4, 4, 4, 2, 1]
    assert chunk_weights(5, taper=8) == [1, 2, 4, 2, 1]
    assert chunk_weights(1, taper=4) == [1]
    w = chunk_weights(64, taper=16)
    assert w == w[::-1] and max(w) == 16 and min(w) == 1
