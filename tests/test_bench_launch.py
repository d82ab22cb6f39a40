"""bench.py's rank launch (CPU, gloo): `--gpus N` outside torchrun re-runs the
script as N ranks under torch.distributed.run, and under torchrun WORLD_SIZE
must equal --gpus (a driver run of `--gpus 8` must not silently
measure one rank)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=env)


def test_gpus_2_starts_two_ranks():
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["gpus_arg"] == 2 and sorted(lines[0]["ranks"]) == [0, 1]


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)


def test_default_is_one_rank():
    r = _run(["--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["n_gpus"] == 1 and line["ranks"] == [0]


def test_reference_arm_runs_cfg4_without_the_product_library():
    """The driver's reference arm (`bench.py --impl reference`, default cfg4):
    one (object, preshape) unit through the unmodified reference
    optimize_grasp on the host cores, inputs from the oracle-side fixture
    library; the process must not map the product libasicp.so."""
    import pytest

    sys.path.insert(0, str(ROOT))
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('MAPS_PRODUCT', 'libasicp.so' in maps, 'libasicp_fixtures.so' in maps)\n")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"].startswith("cfg4")
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "MAPS_PRODUCT False False" in r.stdout
