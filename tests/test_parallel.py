"""Multi-process host logic of the sharded paths on CPU with the
gloo backend, world_size 2: batch sharding + logits gather, and sharded
tuning-trial measurement with a single DB writer."""
import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_04799_b200.parallel import gather_rows, shard_batch, shard_configs, sharded_measure


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        # batch sharding: every rank computes "logits" for its own images
        gb = 7
        start, cnt = shard_batch(gb, ws, rank)
        images = torch.arange(gb, dtype=torch.float32)[start:start + cnt]
        logits = images[:, None] * torch.tensor([1.0, 10.0, 100.0])  # [cnt, 3]
        full = gather_rows(logits, gb)
        # sharded tuning: measure = deterministic cost of the config
        cfgs = [{"tile_n": 64 * (1 + i % 3), "tile_m": 128 * (1 + i % 2)} for i in range(9)]
        seen = []

        def measure(c):
            seen.append(json.dumps(c, sort_keys=True))
            return {"config": c, "cost": c["tile_n"] / c["tile_m"], "rank": rank}
        recs = sharded_measure(cfgs, measure)
        if rank == 0:  # single writer
            with open(os.path.join(out_dir, "trials.jsonl"), "w") as f:
                for r in recs:
                    f.write(json.dumps(r) + "\n")
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump({"full": full.tolist(), "measured": seen}, f)
    finally:
        dist.destroy_process_group()


def test_shard_batch_partitions():
    for gb in (1, 7, 256):
        for ws in (1, 2, 3, 8):
            if gb < ws:
                with pytest.raises(ValueError):
                    shard_batch(gb, ws, 0)
                continue
            parts = [shard_batch(gb, ws, r) for r in range(ws)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == gb
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(ws - 1))
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    assert shard_configs(9, 2, 1) == [1, 3, 5, 7]


def test_gloo_world2_gather_and_sharded_tuning(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "rank0.json"))
    r1 = json.load(open(tmp_path / "rank1.json"))
    want = [[i * 1.0, i * 10.0, i * 100.0] for i in range(7)]
    assert r0["full"] == want and r1["full"] == want  # rank order, uneven split
    # every config measured exactly once across the ranks
    assert len(r0["measured"]) + len(r1["measured"]) == 9
    assert not set(r0["measured"]) & set(r1["measured"])
    lines = [json.loads(l) for l in open(tmp_path / "trials.jsonl")]
    assert [l["config"]["tile_n"] for l in lines] == [64 * (1 + i % 3) for i in range(9)]
    assert {l["rank"] for l in lines} == {0, 1}
