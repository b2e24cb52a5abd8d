"""bench.py's reference arm (the CPU oracle, as the task statement specifies for this tier):
one JSON line with the contract's keys, the same `config` object as our arm, and under
torchrun only rank 0 prints (the other ranks exit 0 without work).  CPU only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--config", "C1", "--steps", "1", "--warmup", "0"],
                          capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)


def test_reference_line():
    p = run({})
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    sys.path.insert(0, ROOT)
    import bench
    import spamm_inputs as si
    cfg = si.CONFIGS["C1"]
    kind, payload = si.make_input(cfg)
    ns = type("A", (), dict(tau=None, iters=None, tau_s_factor=None, t_stop=None, map="plain",
                            channel="dual", partition="equal", dist_world1=False))()
    assert d["config"] == bench.run_config(ns, cfg, 1, bench.payload_bytes(kind, payload))


def test_reference_other_ranks_silent():
    p = run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0, p.stderr
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")]
