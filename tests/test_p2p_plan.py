"""Placement algebra of the peer-memory exchange (csrc/p2p.cu k_plan,
restated by runtime.p2p_plan): simulate one all-to-all-v round trip for
random count matrices and check that every owner receives each source's
keys as one contiguous segment in ascending source order (the order the
owner reduction relies on, reference runtime.py:177-185) and that the
answers come back to each requester in its own send order."""
import numpy as np
import pytest

from paper_1711_06505_b200.runtime import p2p_plan


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seed", [0, 1])
def test_round_trip_placement(world, seed):
    rng = np.random.default_rng(seed)
    cmat = rng.integers(0, 7, (world, world))
    cmat[rng.random((world, world)) < 0.2] = 0  # empty segments
    # send buffers: rank s sends tokens (s, d, i) to owner d, ordered by destination
    send = []
    for s in range(world):
        send.append([(s, d, i) for d in range(world) for i in range(cmat[s, d])])
    recv = [[None] * int(cmat[:, d].sum()) for d in range(world)]
    for s in range(world):
        so, pos, _, _ = p2p_plan(cmat, s)
        for d in range(world):
            seg = send[s][so[d]:so[d + 1]]
            recv[d][pos[d]:pos[d] + len(seg)] = seg
    for d in range(world):
        _, _, ro, _ = p2p_plan(cmat, d)
        assert all(x is not None for x in recv[d])
        for s in range(world):
            assert recv[d][ro[s]:ro[s + 1]] == [(s, d, i) for i in range(cmat[s, d])]
    # answers: owner d returns f(token) for each received token to its requester
    back = [[None] * len(send[s]) for s in range(world)]
    for d in range(world):
        _, _, ro, bp = p2p_plan(cmat, d)
        for s in range(world):
            ans = [("ans",) + t for t in recv[d][ro[s]:ro[s + 1]]]
            back[s][bp[s]:bp[s] + len(ans)] = ans
    for s in range(world):
        assert back[s] == [("ans",) + t for t in send[s]]
