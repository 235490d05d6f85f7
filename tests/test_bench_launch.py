"""bench.py's multi-GPU launch contract, on CPU (no GPU needed).

`--gpus N` without torchrun starts N ranks itself (torch.distributed.run on
127.0.0.1, NCCL_DEBUG=INFO), and refuses to time fewer GPUs than asked.
The rank bodies of `--launch-check` use gloo, so the spawn path runs here.
"""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(REPO, "bench.py")


def run(args, env_extra=None, timeout=300):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT",
                        "NCCL_DEBUG")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=REPO)


def test_launcher_spawns_two_gloo_ranks():
    out = run(["--gpus", "2", "--launch-check"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout          # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2
    assert rec["ranks_mask"] == 0b11            # both ranks joined the all_reduce
    assert rec["master_addr"] == "127.0.0.1"
    assert rec["nccl_debug"] == "INFO"


def test_too_few_gpus_is_an_error():
    out = run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert out.returncode == 2
    assert "needs 2 visible GPUs" in out.stderr
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]


def test_world_size_mismatch_is_an_error():
    out = run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode == 2
    assert "WORLD_SIZE=2" in out.stderr
