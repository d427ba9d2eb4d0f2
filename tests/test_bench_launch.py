"""bench.py's multi-rank launch path on CPU: ``--gpus N`` without a torchrun
environment re-executes itself under torchrun (N ranks, rendezvous on
127.0.0.1, gloo for the dry run), and the reference arm at N ranks times the
same global batch (batch x N) and prints the GPU arm's config dict."""

from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(*argv, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *argv], capture_output=True, text=True,
                       timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return lines[0], r.stderr


def test_gpus_flag_spawns_that_many_ranks():
    line, err = _run("--gpus", "3", "--dry-run")
    assert line["n_gpus"] == 3 and line["max_rank"] == 2 and line["local_world"] == 3
    assert "torch.distributed.run" in err and "--nproc-per-node=3" in err


def test_reference_arm_times_the_global_batch_at_n_ranks():
    line, _ = _run("--gpus", "2", "--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    cfg = line["config"]
    assert cfg["global_batch"] == 2 and cfg["batch_per_gpu"] == 1 and cfg["parallelism"] == "ep2"
    assert "block_widths" not in cfg and "rates" not in cfg  # the executed split is the GPU arm's `split` key
    assert "cc=0.2000 cg=0.3000 gg=0.5000" in line["cpu_baseline"]["sample"]
    assert "2 token(s)" in line["cpu_baseline"]["sample"]
    assert line["cpu_baseline"]["best"] >= line["cpu_baseline"]["median"] > 0
    assert line["cpu_baseline"]["threadpool"]


def test_both_arms_share_one_config_builder():
    """run_ours prints base_config(...) unchanged (the executed split goes under
    `split`, planning detail under `plan` / `calibration`), so the two arms'
    config dicts have the same keys and values."""
    src = (ROOT / "bench.py").read_text()
    assert "config = base_config(args, global_batch, world)" in src
    assert "config.update(" not in src
