"""bench.py's launch contract on CPU: `--gpus N` outside torchrun re-launches itself with N ranks
(torch.distributed.run, 127.0.0.1 rendezvous); under a torchrun environment WORLD_SIZE must equal
--gpus; the reference arm (the CPU oracle) runs on rank 0 only and prints one JSON line with real,
measured steps."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=600, cwd=ROOT)


def test_gpus_2_relaunches_two_ranks_reference_arm():
    r = _run(["--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "3",
              "--cpu-budget", "0.5"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["steps"] == 2
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_world_size_must_match_gpus():
    r = _run(["--impl", "reference", "--gpus", "2", "--config", "1"], env={"WORLD_SIZE": "1"})
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
