"""World-size-2 item sharding on CPU (gloo): the host-side statement of the
multi-GPU path (paper_2510_23264_b200/shard.py; libcqg's NCCL all-reduce of
per-edge partial sums). Each rank scores every edge on its item block with
the oracle, the partial sums are all-reduced over gloo, and the combined mean
must equal the single-process score over all items (proj/src/patching.cpp:
229-238 sums items sequentially in double; the sharded order differs, hence a
1e-12 relative tolerance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import INT8, KL, LOGITDIFF, Policy, Port
from paper_2510_23264_b200 import shard
from helpers import SMALL, TOY, make

RTOL = 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, items, metric, out_path, split=False, mode=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, ds = make(cfg, 1, items, 2)
        p = Port(cfg, w.mats, qkv_split=split)
        lo, hi = shard.item_block(rank, world, items)
        edges = p.sweep_order()
        part = shard.partial_sums(
            p.score_edges(ds.subset(list(range(lo, hi))), edges, Policy.head_quantized(mode=mode),
                          True, metric), hi - lo)
        t = torch.from_numpy(part)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        if rank == 0:
            np.save(out_path, shard.combine(t.numpy(), items))
    finally:
        dist.destroy_process_group()


def test_item_block_partition():
    for items in (1, 2, 5, 64, 255):
        for world in (1, 2, 3, 8):
            blocks = [shard.item_block(r, world, items) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == items
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.item_block(2, 2, 4)


@pytest.mark.parametrize("cfg,items,metric,split,mode", [
    (SMALL, 5, KL, False, 0), (TOY, 4, KL, False, 0), (SMALL, 4, LOGITDIFF, False, 0),
    # the extensions shard the same way: Q/K/V-split graph, INT8 low precision
    (SMALL, 4, KL, True, 0), (TOY, 3, KL, False, INT8)])
def test_two_rank_scores_match_single(tmp_path, cfg, items, metric, split, mode):
    out = str(tmp_path / "combined.npy")
    mp.start_processes(_worker, args=(2, _free_port(), cfg, items, metric, out, split, mode), nprocs=2,
                       join=True, start_method="spawn")
    combined = np.load(out)
    w, ds = make(cfg, 1, items, 2)
    p = Port(cfg, w.mats, qkv_split=split)
    full = p.score_edges(ds, p.sweep_order(), Policy.head_quantized(mode=mode), True, metric)
    assert combined.shape == full.shape
    np.testing.assert_allclose(combined, full, rtol=RTOL, atol=1e-300)
