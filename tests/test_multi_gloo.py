"""N > 1 host logic on CPU: world_size-2 gloo process groups.  Each rank
computes its shard with the CPU oracle (standing in for its GPU), the shards
are gathered, and the result must equal the single-process computation;
max-over-ranks timing is the max of the per-rank values."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import oracle as O
from paper_1901_01965_b200 import shard as SH


def _free_port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def _worker(rank, world, port, n, c_out, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        x, w = synth.random_layer(rng, n, 9, 10, 5, c_out, O.NHWC)
        sh = SH.shard(n, c_out, world, rank)
        xs = x[sh["n0"]: sh["n0"] + sh["n"]]
        ws = w[sh["co0"]: sh["co0"] + sh["co"]]
        if xs.shape[0] and ws.shape[0]:
            local = O.wino_conv(xs, ws, 1, O.NHWC, scaling=True).out32
        else:
            local = np.zeros((xs.shape[0], 9, 10, ws.shape[0]), np.int32)
        full = SH.gather_nhwc(torch.from_numpy(local), (n, 9, 10, c_out), sh, world)
        t = SH.max_over_ranks(float(rank + 1) * 0.5)
        if rank == 0:
            q.put((full.numpy(), t, sh["mode"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,c_out", [(5, 6), (2, 7), (1, 5), (1, 1)])
def test_sharded_equals_single(n, c_out):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, c_out, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, t, mode = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(123)
    x, w = synth.random_layer(rng, n, 9, 10, 5, c_out, O.NHWC)
    np.testing.assert_array_equal(full, O.wino_conv(x, w, 1, O.NHWC, scaling=True).out32)
    assert t == 1.0                        # max over ranks of (0.5, 1.0)
    assert mode == ("batch" if n >= world else "cout")


def test_split_is_a_partition():
    for total in range(0, 20):
        for world in range(1, 9):
            parts = [SH.split(total, world, r) for r in range(world)]
            assert sum(c for _, c in parts) == total
            pos = 0
            for s, c in parts:
                assert s == pos; pos += c


@pytest.mark.parametrize("config,gpus", [("C2", 2), ("C1", 8), ("C5", 2)])
def test_bench_gpus_spawns_ranks_with_their_shards(config, gpus):
    """`bench.py --gpus N` with no WORLD_SIZE re-runs itself under torch.distributed.run with N ranks
    (gloo here, --plan-only: no CUDA); each rank gets its slice of the configured batch (Cout for
    C1's batch 1, where ranks 4-7 of 8 get an empty shard), and the checking gather reassembles the
    full output with every element owned by exactly one rank."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(gpus), "--config", config,
                        "--plan-only"], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["world"] == gpus and line["torchrun"]
    layer = synth.CONFIGS[config].layers[0]
    shards = line["shards"]
    assert len(shards) == gpus
    for rank, sh in enumerate(shards):
        assert sh == SH.shard(layer.n, layer.c_out, gpus, rank)
    ho, wo = layer.h + 2 * layer.pad - 2, layer.w + 2 * layer.pad - 2
    assert line["gathered_shape"] == [layer.n, ho, wo, layer.c_out]
    per_rank = line["elements_per_rank"]
    assert sum(per_rank) == layer.n * ho * wo * layer.c_out
    for rank, sh in enumerate(shards):
        assert per_rank[rank] == sh["n"] * ho * wo * sh["co"]
    if config == "C1":
        assert all(s["mode"] == "cout" for s in shards)
        assert [s["co"] for s in shards] == [1, 1, 1, 1, 0, 0, 0, 0]
    else:
        assert all(s["mode"] == "batch" for s in shards)
    assert line["max_over_ranks"] == 0.25 * gpus
