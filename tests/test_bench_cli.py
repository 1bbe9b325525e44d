"""bench.py's launch contract on CPU: --gpus N outside torch.distributed.run
re-launches itself as N ranks (rank 0 alone prints the reference arm's one
JSON line), and a CK_* override refuses to run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, env=e, timeout=timeout, cwd=ROOT)


def test_gpus_n_relaunches_as_ranks():
    r = _run(["--gpus", "2", "--impl", "reference", "--net", "lenet", "--steps", "1",
              "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2
    assert out["metric"] == "LeNet fwd+bwd images/sec" and out["value"] > 0
    assert out["cpu_baseline"]["kind"] == "reference"


def test_ck_override_refused():
    r = _run(["--steps", "1"], env={"CK_TC_BM": "128"})
    assert r.returncode == 2
    assert "refusing to run" in r.stderr
