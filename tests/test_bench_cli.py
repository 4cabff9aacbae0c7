"""bench.py's driver contract on CPU: the reference arm (the CPU oracle)
prints one JSON line with the contract's keys, simulating G = --gpus ranks
without torchrun (`--impl reference --gpus N` must simulate N)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_simulates_gpus():
    d = _run("--impl", "reference", "--gpus", "2", "--config", "tiny", "--steps", "1",
             "--warmup", "0")
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["G"] == 2
    assert d["config"]["workload"] == "tiny"
    for k in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] == 1


def test_default_headline_is_tieba():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    sys_argv = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = b.parse()
    finally:
        sys.argv = sys_argv
    assert a.config == "tieba" and a.gpus == 1 and a.warmup >= 3
