"""The N>1 path on CPU: world_size-2 gloo process group running the sharding harness
(paper_1407_4859_b200.sharding, used by bench.py under torchrun).  Each rank builds its
contiguous shard as its own layout instance, remaps it (the oracle stands in for the GPU
kernel here -- no GPU on this box), and the union of the shards must equal the
single-process result (record locality).  The timing reduction must
return the max over ranks."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scaling, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from adha_inputs import config_widths, field_columns
        from oracle import remap as O
        from paper_1407_4859_b200.sharding import shard_for, max_over_ranks, aggregate_gbs
        widths = config_widths(16)
        n_cfg = 1001
        n_total, lo, hi = shard_for(n_cfg, world, rank, scaling)
        cols = field_columns(77, n_total, widths)                  # the whole job's records
        mine = [c[lo:hi] for c in cols]
        src = O.pack(mine, widths, [0] * 16, hi - lo)
        dst = np.full(O.layout_bytes(widths, list(range(16)), hi - lo), 0xA5, np.uint8)
        O.remap(src, [0] * 16, dst, list(range(16)), widths, hi - lo)
        got = O.unpack(dst, widths, list(range(16)), hi - lo)
        objs = [None] * world
        dist.all_gather_object(objs, (lo, hi, [g.tobytes() for g in got]))
        ms = max_over_ranks(1.5 + rank)                              # rank r "took" 1.5 + r ms
        dist.barrier()
        if rank == 0:
            q.put((n_total, objs, ms, aggregate_gbs(n_total, 80, 1, 10, ms)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_two_rank_gloo_shards(scaling):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scaling, q)) for r in range(2)]
    for p in procs:
        p.start()
    n_total, objs, ms, gbs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from adha_inputs import config_widths, field_columns
    widths = config_widths(16)
    assert n_total == (2002 if scaling == "weak" else 1001)
    # contiguous, covering, balanced shards
    (lo0, hi0, s0), (lo1, hi1, s1) = objs
    assert lo0 == 0 and hi0 == lo1 and hi1 == n_total and abs((hi0 - lo0) - (hi1 - lo1)) <= 1
    cols = field_columns(77, n_total, widths)
    for f, w in enumerate(widths):
        union = np.frombuffer(s0[f] + s1[f], np.uint8).reshape(-1, w)
        assert np.array_equal(union, cols[f])                          # shard union == 1-process result
    assert ms == 2.5                                                   # max over ranks
    assert gbs == pytest.approx(2 * n_total * 80 * 10 / 2.5e-3 / 1e9)


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the CPU oracle on the bench workload) prints one valid JSON line
    with the contract's keys; no GPU needed."""
    import json
    import subprocess
    import sys
    from tests.conftest import ROOT
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
