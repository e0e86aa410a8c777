"""Batch sharding of bench.py for configs 2-4 (weak scaling, no collective in
the solve): rank r of world W solves the signals [rB, (r+1)B), each seeded by
its GLOBAL index, so the union over ranks is exactly the single-process batch
of W*B signals.  Checked with two gloo ranks on CPU (host generation only)."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, cfgn, B, q):
    sys.path.insert(0, ROOT)
    import torch
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.CFG.clear()
    bench.CFG.update(bench.CONFIGS[cfgn])
    rows, Y, tol = bench.problem(B, rank * B)
    Yc = np.ascontiguousarray(Y.astype(np.complex128))
    yt = torch.from_numpy(Yc.view(np.float64).copy())
    tt = torch.from_numpy(np.ascontiguousarray(tol))
    ys = [torch.empty_like(yt) for _ in range(world)]
    ts = [torch.empty_like(tt) for _ in range(world)]
    dist.all_gather(ys, yt)
    dist.all_gather(ts, tt)
    if rank == 0:
        _, Yall, tall = bench.problem(world * B, 0)
        got = np.concatenate([y.numpy() for y in ys]).view(np.complex128)
        q.put(bool(np.array_equal(got, Yall.astype(np.complex128))) and
              bool(np.array_equal(np.concatenate([t.numpy() for t in ts]), tall)))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfgn,B", [(2, 6), (4, 3)])
def test_bench_shards_union_is_the_global_batch(cfgn, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 37 * cfgn + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfgn, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("scaling,firsts,per", [("weak", [0, 4096], 4096), ("strong", [0, 2048], 2048)])
def test_bench_gpus2_launches_two_ranks(scaling, firsts, per):
    """`bench.py --gpus 2` without a launcher starts two ranks itself (gloo in
    the dry run: no GPU here), shards by global signal index and reports the
    world size it actually ran."""
    import json
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "2", "--warmup", "3", "--scaling", scaling],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["rank_first_signal"] == firsts and line["batch_per_gpu"] == per
    assert line["scaling"] == scaling and line["config"]["batch"] == 4096


def test_bench_rejects_mismatched_world_size():
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 2


@pytest.mark.parametrize("cfgn", [1, 2, 4])
def test_reference_arm_inputs_without_the_cuda_package(cfgn):
    """The reference arm's inputs come from the reference's own generators
    (oracle library): the harness's inputs up to the last bits of y, and the
    process never loads the CUDA package."""
    import subprocess
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import bench
bench.CFG.update(bench.CONFIGS[{cfgn}])
orc, kind = bench.reference_oracle()
rows, Y, tol = bench.problem_oracle(orc, 3, 5)
maps = open('/proc/self/maps').read()
print(int('libfmp_cuda' in maps), int('paper_1205_4139_b200' in sys.modules))
np.save(sys.argv[1], np.concatenate([Y.astype(np.complex128).ravel(), tol.astype(np.complex128)]))
"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "v.npy")
        out = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True,
                             timeout=300, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-2000:]
        assert out.stdout.split() == ["0", "0"]
        v = np.load(f)
    sys.path.insert(0, ROOT)
    import bench
    bench.CFG.clear()
    bench.CFG.update(bench.CONFIGS[cfgn])
    _, Y, tol = bench.problem(3, 5)
    w = np.concatenate([Y.astype(np.complex128).ravel(), tol.astype(np.complex128)])
    # the draws are identical; y = Phi x + e is synthesised by the reference
    # through its transform and by the host generator as direct sums over the
    # K nonzeros, so y differs in the last bits
    assert np.allclose(v, w, rtol=1e-12, atol=1e-14 * np.abs(w).max())
