"""Multi-rank host logic of the batch-sharded path on CPU:
world_size 2 over gloo.  The GPU kernels are replaced by the CPU oracle here
(this is a test — the oracle is the checker); what is under test is the
sharding, per-signal-seed reproducibility of shards, max-over-ranks timing
and the verification gathers the bench performs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16665_b200.dist import gather_checksums, gather_shards, max_over_ranks, shard_range


def test_shard_range_partitions_batch():
    for total in (0, 1, 7, 8, 65536, 65537):
        for ws in (1, 2, 3, 4, 8):
            spans = [shard_range(total, ws, r) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import alpha_oracle as orc
        from paper_2403_16665_b200.signals import WORKLOADS, generate

        w = WORKLOADS["4"]
        lo, hi = shard_range(total, world, rank)
        x = generate(w, lo, hi - lo, threads=1)  # this rank's shard only, per-signal seeds
        out = torch.from_numpy(orc.alpha_fft(x.astype(np.complex128)[:, :256], 1, 8, 256))
        full = gather_shards(out, total)
        t = max_over_ranks(float(rank + 1))
        chk = gather_checksums(out)
        q.put((rank, full.numpy(), t, chk))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_reproduce_single_process():
    total, world = 5, 2  # ragged: shards of 3 and 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import alpha_oracle as orc
    from paper_2403_16665_b200.signals import WORKLOADS, generate

    x = generate(WORKLOADS["4"], 0, total, threads=1)
    want = orc.alpha_fft(x.astype(np.complex128)[:, :256], 1, 8, 256)
    for rank, full, t, chk in results:
        assert full.shape == want.shape
        np.testing.assert_array_equal(full, want)  # shards are independent and exact
        assert t == 2.0  # job time = slowest rank
        assert len(chk) == 2
