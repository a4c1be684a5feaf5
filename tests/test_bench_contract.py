"""bench.py's JSON contract on the CPU: the reference arm (the compiled reference / the oracle on
the host cores) runs without a GPU, so its line — and with it the keys both arms share — is
checked here on the small config C1; the GPU arm's line is checked by the driver on a B200."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_schema():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("CoR-UTV decomps/sec") and line["unit"] == "decomps/s"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    assert line["higher_is_better"] is True and line["data"] == "synthetic" and line["dtype"] == "f64"
    assert line["value"] > 0 and abs(line["value"] - 1e3 / line["ms_per_step"]) <= 1e-6 * line["value"]
    cfg = line["config"]
    assert cfg["workload"].startswith("C1:") and "model" not in cfg
    assert len(cfg["a_sha256"]) == 64 and cfg["phi"].startswith("host-exact")
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "decomps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_gpus_flag_without_devices_fails_loudly():
    """--gpus 2 outside torchrun must not silently run one rank: with fewer visible
    GPUs than asked for it exits non-zero with a message."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert p.returncode != 0
    assert "--gpus 2" in (p.stderr + p.stdout)
