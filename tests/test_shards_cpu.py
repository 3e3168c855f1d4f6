"""CPU: the substrate x z-slab layout logic (which rank holds which
substrates and planes) — no device needed."""
import pytest

from paper_2110_13368_b200.shards import layout_for, rank_piece, split_substrates


def test_layout_defaults_prefer_substrate_shards():
    assert layout_for(1, 4, 1024) == (1, 1)
    assert layout_for(2, 4, 1024) == (2, 1)
    assert layout_for(4, 4, 1024) == (4, 1)
    assert layout_for(8, 4, 1024) == (4, 2)
    assert layout_for(8, 2, 1024) == (2, 4)
    assert layout_for(6, 4, 1024) == (2, 3)
    assert layout_for(8, 4, 1024, substrate_parts=1) == (1, 8)
    with pytest.raises(ValueError):
        layout_for(8, 4, 1024, substrate_parts=3)
    with pytest.raises(ValueError):
        layout_for(8, 1, 4)


def test_rank_pieces_tile_the_problem_once():
    for world, S, nz, k in [(8, 4, 64, None), (8, 4, 64, 2), (6, 3, 30, None), (4, 4, 9, 1)]:
        cells = set()
        for r in range(world):
            (s0, s1), (z0, z1), slab, P, shard = rank_piece(r, world, S, nz, k)
            assert 0 <= slab < P and shard * P + slab == r
            for s in range(s0, s1):
                for z in range(z0, z1):
                    assert (s, z) not in cells
                    cells.add((s, z))
        assert len(cells) == S * nz


def test_split_substrates_errors():
    with pytest.raises(ValueError):
        split_substrates(2, 3)
    assert split_substrates(4, 3) == [(0, 1), (1, 3), (3, 4)]
