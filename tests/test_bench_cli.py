"""bench.py's launch contract on the CPU box (no GPU needed): the reference
arm prints one JSON line with the contract's keys, and `--gpus N` outside a
torchrun environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1 rendezvous), of which rank 0 alone prints."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *map(str, args)], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    return lines


@pytest.mark.parametrize("gpus", [1, 2])
def test_reference_arm_contract_and_self_launch(gpus):
    lines = _bench("--impl", "reference", "--gpus", gpus, "--config", 1, "--steps", 20, "--warmup", 10)
    assert len(lines) == 1, lines  # rank 0 only
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == gpus
    assert d["metric"] == "fp64 Laplacian matvecs/sec" and d["unit"] == "matvecs/s" and d["higher_is_better"]
    assert d["value"] > 0 and d["config"]["workload"] == "config1"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
