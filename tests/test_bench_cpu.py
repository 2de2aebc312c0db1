"""bench.py contract on CPU: the multi-GPU launcher, the shared config of the
two arms, and the reference arm running the unmodified reference."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, env=e, cwd=str(ROOT))


def test_gpus_flag_fails_loudly_without_enough_devices():
    """--gpus N outside torchrun re-launches N ranks; with fewer visible GPUs
    (here none) it exits non-zero with the reason instead of timing 1 rank."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs: the launcher would really run")
    p = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=300)
    assert p.returncode == 2
    assert "--gpus 2 requested" in p.stderr


def test_world_size_must_match_gpus():
    p = _run(["--gpus", "1"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"},
             timeout=300)
    assert p.returncode == 2 and "WORLD_SIZE=2" in p.stderr


def test_both_arms_share_the_config_object():
    sys.path.insert(0, str(ROOT))
    import bench
    args = bench.parse(["--config", "cfg2", "--gpus", "2"])
    _scene, views, desc, _ = bench.workload("cfg2", 2)
    assert len(views) == 16                      # weak scaling: 8 views per rank
    cfg = bench.config_of(args, 2, desc)
    assert cfg["scaling"] == "weak" and cfg["parallelism"].startswith("anchor-sharded x2")
    assert cfg["views_per_step"] == 16
    assert bench.CITY["cfg3"][5] == "strong" and bench.CITY["cfg4"][3:5] == (3840, 2160)


@pytest.mark.slow
def test_reference_arm_runs_the_unmodified_reference():
    sys.path.insert(0, str(ROOT))
    import bench
    if not bench.reference_available():
        from oracle.build_ref import build
        if not build():
            pytest.skip("no oracle/_ref and no /root/reference to install it from")
    p = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-tiles", "4",
              "--ref-cfg1-threads", ""], timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert "UNMODIFIED reference" in line["cpu_baseline"]["sample"]
    assert line["config"]["parallelism"] == "single" and line["config"]["scaling"] == "weak"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
