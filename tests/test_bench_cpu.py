"""bench.py's reference arm runs on CPU (the reference's own query path from
oracle/_ref): its JSON line carries the contract's keys.  The GPU arm's line
is exercised on the GPU box by the round-end bench run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "1",
                        "--warmup", "1", "--cpu-sample", "32"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "q-grams/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("shard", ["replicas", "blocks"])
def test_bench_gpus_2_spawns_ranks(shard):
    """`bench.py --gpus 2` with no launcher re-runs itself under
    torch.distributed.run with two ranks (the world size is checked against
    --gpus, timing is the max over ranks); the JSON line says n_gpus 2.  The
    CPU oracle stands in for the per-rank engine (--engine oracle, gloo), so
    this tests the launch and the block-shard hit-list exchange, not speed."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--engine", "oracle", "--shard", shard,
                        "--c5-docs", "600", "--c5-block-size", "128", "--c5-median", "3000",
                        "--queries", "6"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["shard"] == shard and d["value"] > 0
    if shard == "blocks":
        assert d["hits_identical"] is True


def test_bench_world_size_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--engine", "oracle"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_loads_no_product_library():
    """--impl reference must not load the product library (or any library
    outside oracle/): its inputs come from the oracle's copy of the seeded
    generator.  Checked from /proc/self/maps at exit."""
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', "
            "'--warmup', '0', '--cpu-sample', '8'];\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    maps = [l for l in r.stdout.splitlines() if l.startswith("MAPS")][0]
    repo_libs = [x for x in eval(maps[5:]) if x.startswith(ROOT)]
    assert repo_libs and all(x.startswith(os.path.join(ROOT, "oracle")) for x in repo_libs), repo_libs
