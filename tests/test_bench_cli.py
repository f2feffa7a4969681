"""bench.py's multi-rank plumbing without a GPU: `--gpus N` outside torchrun
re-launches itself as N ranks (torch.distributed.run, 127.0.0.1) and the
ranks shard the ResNet-18 global batch, reduce the max time and gather the
logits over gloo -- the same path the 8-GPU run takes over NCCL."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_spawns_eight_gloo_ranks():
    j = _run("--gpus", "8", "--cpu-dry-run", "--steps", "2")
    assert j["n_gpus"] == 8 and j["ranks"] == list(range(8))
    assert j["gathered_rows"] == 256 and j["global_batch"] == 256


def test_bench_refuses_untested_knob_file(tmp_path):
    p = tmp_path / "k.json"
    p.write_text("{}")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--knobs-in", str(p)],
                         capture_output=True, text=True, timeout=600, cwd=REPO,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert out.returncode != 0
    assert "parity tests cover" in (out.stderr + out.stdout)
