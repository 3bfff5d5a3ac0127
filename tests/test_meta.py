"""K8 segment-index builder (csrc/meta.cpp via the C-ABI) vs the reference's
offset semantics (lorapack.py:146-150) -- bit-exact."""

import numpy as np
import pytest

from oracle import lorapack_oracle as O
from paper_2508_02932_b200.meta import build_meta


def test_reference_offset_goldens():
    # pkg/tests/test_lorapack.py:29-35 and :37-46
    m = build_meta([3], [2], [1.0])
    assert m.rank_offsets == (0, 3) and m.row_offsets == (0, 2)
    m = build_meta([8, 16], [3, 2], [1.0, 1.0])
    assert m.rank_offsets == (0, 8, 24) and m.row_offsets == (0, 3, 5)
    assert all(type(v) is int for v in m.rank_offsets + m.row_offsets)


def test_golden_offsets_bit_exact(golden_cases):
    for name, c in golden_cases:
        ranks = np.diff(c["rank_offsets"])
        toks = np.diff(c["row_offsets"])
        m = build_meta(ranks, toks, c["alphas"])
        assert m.rank_offsets == c["rank_offsets"], name
        assert m.row_offsets == c["row_offsets"], name


def _check_tiles(m):
    so = m.row_offsets
    covered = np.zeros(m.total_tokens, dtype=np.int32)
    for m0, ln, a, z in m.mtiles:
        assert z == 0 and 1 <= ln <= 128
        assert so[a] <= m0 and m0 + ln <= so[a + 1]   # never straddles two segments
        covered[m0:m0 + ln] += 1
    assert (covered == 1).all()
    covered[:] = 0
    for m0, ln, a, z in m.ptiles:
        assert z == 0 and 1 <= ln <= 256
        assert so[a] <= m0 and m0 + ln <= so[a + 1]
        covered[m0:m0 + ln] += 1
    assert (covered == 1).all()


def test_random_packs_match_oracle_prefix_sums():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 40))
        ranks = rng.integers(1, 130, n)
        toks = rng.integers(0, 700, n)
        m = build_meta(ranks, toks, np.ones(n))
        assert m.rank_offsets == O.prefix_offsets(ranks)
        assert m.row_offsets == O.prefix_offsets(toks)
        assert np.array_equal(m.token_adapter, O.token_adapter_ids(m.row_offsets))
        rp = (ranks + 15) // 16 * 16
        assert np.array_equal(m.rpad_off, np.concatenate([[0], np.cumsum(rp)]))
        assert m.nb == (int(ranks.max()) + 63) // 64
        _check_tiles(m)


def test_empty_segments_and_rank_zero():
    m = build_meta([4, 2, 9], [0, 5, 0], [1.0, 2.0, 3.0])
    assert m.row_offsets == (0, 0, 5, 5)
    assert m.mtiles.tolist() == [[0, 5, 1, 0]]
    with pytest.raises(ValueError, match="strictly increasing"):
        build_meta([4, 0], [1, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="nothing to pack"):
        build_meta([], [], [])


def test_bench_config_tiles():
    # C3: 16 adapters, b_i * 1024 tokens -> every tile full and single-adapter
    b = [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]
    m = build_meta([8, 16, 32, 64] * 4, [x * 1024 for x in b], [1.0] * 16)
    assert m.total_tokens == 32768
    assert len(m.mtiles) == 256 and (m.mtiles[:, 1] == 128).all()
    assert len(m.ptiles) == 128 and (m.ptiles[:, 1] == 256).all()
