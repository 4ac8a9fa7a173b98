"""Host logic of the rank decomposition (paper_2211_00705_b200.decomp): tile-aligned slicing and
the halo / CFL-pair exchange over a world_size-2 gloo group on CPU."""
import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_00705_b200 import decomp as D  # noqa: E402
from paper_2211_00705_b200 import (HALO, XB_DOUBLES, XB_DT, XB_REC, XB_RECV_LEFT, XB_RECV_RIGHT,  # noqa: E402
                                   XB_SEND_LEFT, XB_SEND_RIGHT)


@pytest.mark.parametrize("n,tile", [(1 << 27, 960), (38917, 960), (9605, 960), (1000, 64), (4096, 1024)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_rank_slices_partition_whole_tiles(n, tile, world):
    T = D.tile_count(n, tile)
    if T < world:
        with pytest.raises(ValueError):
            D.rank_slice(n, tile, 0, world)
        return
    cuts = [D.rank_slice(n, tile, r, world) for r in range(world)]
    assert cuts[0][0] == 0 and cuts[-1][1] == n
    for (a0, a1), (b0, b1) in zip(cuts, cuts[1:]):
        assert a1 == b0 and a1 % tile == 0
    sizes = [c1 - c0 for c0, c1 in cuts]
    assert min(sizes) >= HALO and max(sizes) - min(sizes) <= 2 * tile


def test_tile_count_tiny_remainder():
    assert D.tile_count(960 * 5 + HALO - 1, 960) == 5      # remainder folded into the last tile
    assert D.tile_count(960 * 5 + HALO, 960) == 6
    assert D.tile_count(5, 960) == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        x = torch.full((XB_DOUBLES,), -1.0, dtype=torch.float64)
        x[XB_SEND_LEFT:XB_SEND_LEFT + XB_REC] = torch.arange(XB_REC, dtype=torch.float64) + 1000 * rank + 100
        x[XB_SEND_RIGHT:XB_SEND_RIGHT + XB_REC] = torch.arange(XB_REC, dtype=torch.float64) + 1000 * rank + 500
        x[XB_DT] = -10.0 - rank          # -S_max: the min picks the largest speed
        x[XB_DT + 1] = 5.0 - rank * 0.5   # h_min
        D.exchange_halos(x, rank, world)
        q.put((rank, x.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_halos_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ar = torch.arange(XB_REC, dtype=torch.float64)
    for r in range(world):
        x = torch.tensor(got[r], dtype=torch.float64)
        if r > 0:   # left neighbour's send_right
            assert torch.equal(x[XB_RECV_LEFT:XB_RECV_LEFT + XB_REC], ar + 1000 * (r - 1) + 500)
        else:
            assert torch.all(x[XB_RECV_LEFT:XB_RECV_LEFT + XB_REC] == -1.0)
        if r < world - 1:   # right neighbour's send_left
            assert torch.equal(x[XB_RECV_RIGHT:XB_RECV_RIGHT + XB_REC], ar + 1000 * (r + 1) + 100)
        else:
            assert torch.all(x[XB_RECV_RIGHT:XB_RECV_RIGHT + XB_REC] == -1.0)
        assert x[XB_DT].item() == -10.0 - (world - 1)
        assert x[XB_DT + 1].item() == 5.0 - (world - 1) * 0.5
