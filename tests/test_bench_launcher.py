"""bench.py's multi-GPU launch path on CPU (gloo): `--gpus N` outside torchrun
re-launches itself under torch.distributed.run with N ranks; each rank reads
RANK / WORLD_SIZE / LOCAL_RANK, joins the process group, receives rank 0's NCCL
unique id and builds its share of the partition -- everything up to the first
CUDA call (--dry-run).  Mirrors the reference runner's one-rank-per-worker launch
(proj/src/runner.cpp:189-293)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.parametrize("mesh,extra", [("tgv", ["--elems", "6"]), ("tgv", ["--strong", "--elems", "12"]), ("rotor", [])])
def test_two_rank_launch_up_to_the_first_cuda_call(mesh, extra):
    lines = sorted(run("--gpus", "2", "--dry-run", "--mesh", mesh, *extra), key=lambda d: d["rank"])
    assert [d["rank"] for d in lines] == [0, 1] and all(d["world"] == 2 for d in lines)
    assert [d["local_rank"] for d in lines] == [0, 1]
    assert all(d["nccl_id_bytes"] == 128 for d in lines)
    conf = lines[0]["config"]
    assert sum(d["elements"] for d in lines) == conf["elements"]
    assert all(d["halo_peers"] == [1 - d["rank"]] for d in lines)
    assert all(d["interior_run"][0] == 0 and d["interior_run"][1] > d["elements"] // 2 for d in lines)
    if mesh == "rotor" or "--strong" in extra:  # theta / y slabs of one mesh: equal shares, strong scaling
        assert lines[0]["elements"] == lines[1]["elements"]
        assert conf["scaling"] == "strong"
    if "--strong" in extra:  # the whole mesh is --elems^3, not --elems^3 per GPU
        assert conf["elements"] == 12 ** 3


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 1" in r.stderr
