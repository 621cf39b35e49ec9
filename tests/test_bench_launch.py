"""bench.py's launcher and JSON contract pieces (CPU): ``--gpus N`` without a
torchrun environment re-launches itself with N ranks (gloo here), and both
arms print the same ``config`` object."""

import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_flag_spawns_that_many_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--probe-launch"],
                       capture_output=True, text=True, env=env, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2
    assert sorted(x["rank"] for x in lines[0]["ranks"]) == [0, 1]
    assert len({x["pid"] for x in lines[0]["ranks"]}) == 2


def test_mismatched_world_size_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--probe-launch"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_default_config_is_the_largest_single_gpu_config():
    args = bench.parse([])
    assert args.config == "5" and bench.SHAPES["5"] == (32768, 32768)


def test_both_arms_share_the_config_object():
    for cfg in bench.CONFIGS:
        for world in (1, 2, 8):
            c = bench.bench_config(cfg, world)
            assert c == bench.bench_config(cfg, world)
            assert c["image"] == list(bench.SHAPES[cfg])
    assert bench.bench_config("4", 8)["images_per_rank_per_step"] == 8
    assert "row bands" in bench.bench_config("5", 4)["parallelism"]
