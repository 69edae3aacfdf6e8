"""Multi-rank host logic on the CPU (gloo, world size 2): weak-scaling shards,
max-over-ranks timing, and the reference arm's rank behaviour (DESIGN.md s.7)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle
    import synth
    first = bench.shard_first_index(rank, n)
    x = synth.fill_numpy(2, 1, n, first=first)
    h, p, _ = oracle.batch_sample(oracle.CAP, *[x[k] for k in synth.PLANES], threads=1)
    out = torch.from_numpy(np.vstack([h, p[None]]))
    gathered = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(gathered, out)
    t = bench.reduce_max(float(rank + 1) * 1.5, world)
    if rank == 0:
        q.put((torch.cat(gathered, dim=1).numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_weak_scaling_shards_and_max_over_ranks(orc):
    import synth
    n, world = 4096, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the union of the shards equals one process over 2n samples
    x = synth.fill_numpy(2, 1, world * n)
    h, p, _ = orc.batch_sample(orc.CAP, *[x[k] for k in synth.PLANES], threads=1)
    np.testing.assert_array_equal(got, np.vstack([h, p[None]]))
    assert t == 3.0  # max over ranks of (rank + 1) * 1.5


def test_reference_arm_rank_behaviour():
    """Under torchrun the reference arm runs on rank 0 only; other ranks exit 0."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == ""
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True)
    assert r.returncode == 0
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_shard_recipe_is_index_pure():
    """Counter-based inputs: a sample depends only on its global index."""
    import synth
    a = synth.fill_numpy(5, 4, 1000, first=123456)
    b = synth.fill_numpy(5, 4, 3000, first=122456)
    for k in synth.PLANES:
        np.testing.assert_array_equal(a[k], b[k][1000:2000])
