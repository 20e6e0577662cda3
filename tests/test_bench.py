"""bench.py contract checks that need no GPU: the reference arm maps only the
reference library (never this repo's CUDA library), both arms describe the
workload with the same config dict, the self-check gate refuses a corrupted
weight (bench.cpp:140-167 + the --inject-fault hook, tests/CMakeLists.txt:32-36),
and --gpus is honoured."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=e, cwd=ROOT, timeout=600)


def _need_ref():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built here")


def test_reference_arm_maps_no_repo_library():
    _need_ref()
    code = ("import runpy,sys\n"
            "sys.argv=['bench.py','--impl','reference','--steps','3','--warmup','3','--cpu-images','2',"
            "'--config','c2-b1']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') if '.so' in l and "
            "('/root/repo' in l or 'paper_1911' in l or 'oracle' in l)}))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.splitlines()[0])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    maps = [m for m in r.stdout.splitlines() if m.startswith("MAPS")][0]
    assert "libspcv_cu" not in maps and "libspcv_b200" not in maps
    assert "libspcv_ref.so" in maps


def test_both_arms_share_the_config_dict():
    _need_ref()
    import bench
    from paper_1911_09723_b200.workloads import CONFIGS

    for n in (1, 2, 8):
        r = _run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-images", "1", "--gpus", str(n)])
        assert r.returncode == 0, r.stderr
        line = json.loads(r.stdout.splitlines()[0])
        args = bench.parse_args(["--gpus", str(n)])
        args.global_batch = CONFIGS[args.config]["images"]
        imgs, scaling = bench.rank_images(args, n, 0)
        assert line["config"] == bench.bench_config(args, CONFIGS[args.config]["layers"](), n, imgs)
        assert line["n_gpus"] == n and line["scaling"] == scaling == "strong"
        assert line["config"]["global_batch"] == 256 and line["config"]["images_per_gpu"] == 256 // n


def test_selfcheck_gate_refuses_a_corrupted_weight():
    _need_ref()
    r = _run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-images", "1", "--inject-fault"])
    assert r.returncode == 2
    assert r.stdout.strip() == ""  # no JSON line
    assert "refusing to emit records" in r.stderr


def test_gpus_must_match_world_size():
    r = _run(["--gpus", "2", "--steps", "3"], env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_strong_shards_tile_the_global_batch():
    import bench

    args = bench.parse_args(["--gpus", "8"])
    args.global_batch = 256
    sizes = [bench.rank_images(args, 8, r)[0] for r in range(8)]
    assert sizes == [32] * 8
    args.global_batch = 13
    assert sum(bench.rank_images(args, 4, r)[0] for r in range(4)) == 13
    args.images_per_gpu = 256
    assert bench.rank_images(args, 8, 3) == (256, "weak")


def test_l2_flush_chosen_for_small_working_sets():
    import bench
    from paper_1911_09723_b200.workloads import CONFIGS

    args = bench.parse_args([])
    for name, flushed in (("c1", True), ("c2-b1", True), ("c2-b256", False), ("c5", False)):
        args.config = name
        args.global_batch = CONFIGS[name]["images"]
        cfg = bench.bench_config(args, CONFIGS[name]["layers"](), 1, CONFIGS[name]["images"])
        assert ("flushed" in cfg["l2"]) == flushed, (name, cfg["l2"])
