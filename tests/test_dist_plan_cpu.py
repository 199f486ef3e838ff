"""The row-sharded symmetric apply's tile plan (liblaker.so's host planner, called through
laker_debug_dist_tiles -- no GPU needed).  K = exp(scale E E^T) is symmetric (P:141-147
with q = k, reading R2), so every entry pair K_ij = K_ji must be streamed exactly once
over all ranks: as a row contribution K_ij x_j to y_i of the tile's block-row, and,
for a tile off the diagonal block, as the column contribution K_ij x_i to y_j.  The
plan must cover every ordered (i, j) exactly once, give every rank n^2 / (2 W) entries,
and list for each column tile the local block-rows holding its column partials."""
import numpy as np
import pytest

BR, TC = 128, 64


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.mark.parametrize("TC", [64, 128])     # the fp64 kernel's 128 x 64 tiles, the tensor-core 128 x 128
@pytest.mark.parametrize("n,W", [(1024, 1), (2048, 2), (3072, 3), (2048, 4), (2560, 5), (4096, 8), (1536, 6), (7168, 7)])
def test_plan_covers_each_entry_once_and_balances(L, n, W, TC):
    R = BR // TC                      # column sub-blocks per tile row block
    nsb = n // TC                     # TC-wide sub-blocks: a tile is R x 1 of them
    count = np.zeros((nsb, nsb), dtype=np.int64)
    tiles = []
    for w in range(W):
        p = L.laker_debug_dist_tiles(n, BR, TC, w, W)
        toff, jt, lo, hi = p["toff"], p["jt"], p["cr_lo"], p["cr_hi"]
        Lb = len(toff) - 1
        assert Lb == n // W // BR
        cols = {}
        for I in range(Lb):
            Ig = w * Lb + I
            for j in jt[toff[I]:toff[I + 1]]:
                for rsb in range(R * Ig, R * Ig + R):
                    count[rsb, j] += 1               # row contribution K_ij x_j -> y_i
                    if j // R != Ig:
                        count[j, rsb] += 1           # column contribution K_ij x_i -> y_j
                if j // R != Ig:
                    cols.setdefault(int(j), set()).add(I)
        for j in range(nsb):
            have = cols.get(j, set())
            assert have == set(range(lo[j], hi[j])), (w, j, sorted(have), lo[j], hi[j])
        tiles.append(int(toff[-1]))
    assert (count == 1).all(), np.argwhere(count != 1)[:5]
    # balance: each rank streams the single-GPU triangle / W, in tiles of BR x TC
    per = (n // W) ** 2 * W / 2 / (BR * TC)
    assert all(abs(t - per) <= n // W // BR for t in tiles), (tiles, per)
    # W = 1 is the single-GPU plan: block-row I streams column tiles R I .. n/TC - 1
    if W == 1:
        p = L.laker_debug_dist_tiles(n, BR, TC, 0, 1)
        exp = np.concatenate([np.arange(R * I, nsb) for I in range(n // BR)])
        assert (p["jt"] == exp).all()


@pytest.mark.parametrize("n,W", [(1000, 2), (2048, 3), (1536, 4)])
def test_plan_rejects_unaligned_shards(L, n, W):
    with pytest.raises(L.LakerError):
        L.laker_debug_dist_tiles(n, BR, TC, 0, W)
