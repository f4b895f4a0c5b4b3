"""bench.py's host-side contract, on CPU: the reference arm's JSON line (it
times the reference's own CPU path -- numba from baseline/_ref when it is
installed, else the C restatement) and the refusal of a torchrun world that
contradicts --gpus."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_line_keys():
    r = _run(["--impl", "reference", "--cells", "10", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "assembled elements/s" and line["unit"] == "elem/s"
    assert line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["value"] > 0 and line["dtype"] == "f64"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "elem/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["box_cells"] == [10, 10, 10]


def test_mismatched_world_is_refused():
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "0"],
             env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"}, timeout=120)
    assert r.returncode != 0
    assert "refusing a mismatched run" in (r.stderr + r.stdout)
