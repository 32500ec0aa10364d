"""CPU restatement of two tile orders of the grouped GEMM's decode_tile
(paper_2505_11432_b200/csrc/gemm_sm100.cuh), checked for the properties the
kernels rely on:
  - fused TP GEMM-RS order (rs_order): a permutation of all tiles; on every
    rank, the tiles a peer must deliver for one of this rank's own tiles come
    D blocks earlier in that peer's own order (and in-order claims make the
    waits deadlock-free: every awaited tile is claimed before the waiter's);
  - split_last: the last S pair tiles become 2 S half tiles covering the same
    rows exactly once."""
import itertools

import pytest


def rs_order(n, tps, n_tiles, D, self_rank):
    """Sequence of (m-tile, column, own) as decode_tile's rs_order branch."""
    mt, P = n * tps, (n - 1) * tps
    out = []
    for li in range(mt * n_tiles):
        if li < D * P:
            c, r, own = li // P, li % P, False
        elif li < D * P + (n_tiles - D) * (P + tps):
            l2 = li - D * P
            c, r = D + l2 // (P + tps), l2 % (P + tps)
            own = r >= P
            if own:
                r, c = r - P, c - D
        else:
            l3 = li - D * P - (n_tiles - D) * (P + tps)
            c, r, own = n_tiles - D + l3 // tps, l3 % tps, True
        m = self_rank * tps + r if own else ((self_rank + 1) * tps + r) % mt
        out.append((m, c, own))
    return out


@pytest.mark.parametrize("n,tps,n_tiles,D", [(4, 8, 32, 6), (4, 4, 4, 3), (2, 4, 4, 3), (8, 2, 3, 2),
                                             (4, 8, 32, 0), (16, 1, 8, 6)])
def test_rs_order_is_a_permutation_and_peers_deliver_first(n, tps, n_tiles, D):
    D = max(0, min(D, n_tiles - 1))
    orders = [rs_order(n, tps, n_tiles, D, r) for r in range(n)]
    for o in orders:
        assert sorted((m, c) for m, c, _ in o) == sorted(itertools.product(range(n * tps), range(n_tiles)))
    pos = [{(m, c): i for i, (m, c, _) in enumerate(o)} for o in orders]
    for owner, o in enumerate(orders):
        for i, (m, c, own) in enumerate(o):
            assert own == (m // tps == owner)
            if not own:
                continue
            # every peer reaches this tile (its push to `owner`) no later than the
            # owner reaches it: claims are in order on every rank, so the peer's
            # tile is never behind a wait on the owner's side
            for q in range(n):
                if q != owner:
                    assert pos[q][(m, c)] <= i, (owner, q, m, c)


def split_last(total, S):
    """decode_tile's split_last: tile t -> (full tile index, half or None)."""
    out = []
    for t in range(total + S):
        if S > 0 and t >= total - S:
            u = t - (total - S)
            out.append((total - S + u // 2, u & 1))
        else:
            out.append((t, None))
    return out


@pytest.mark.parametrize("total,units", [(320, 74), (96, 74), (32, 74), (12, 74), (1024, 74)])
def test_split_last_covers_every_row_once(total, units):
    rem = total % units
    S = rem if rem > 0 and 2 * rem <= units else 0
    seq = split_last(total, S)
    rows = []
    for t, half in seq:
        base = t * 256
        rows += list(range(base, base + 256)) if half is None else list(range(base + 128 * half, base + 128 * half + 128))
    assert sorted(rows) == list(range(total * 256))
    # the tail wave is at most one round of half tiles
    assert 2 * S <= units
