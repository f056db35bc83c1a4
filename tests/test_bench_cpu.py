"""bench.py contract checks that need no GPU: the reference arm (the oracle,
timed on the host cores) prints one JSON line with the contract's keys, on
the same metric / unit / config as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--config", "qwen3-8b_b32_ctx32k"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "us/step" and d["higher_is_better"] is False
    assert d["config"]["workload"] == "qwen3-8b_b32_ctx32k" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def _launch_check(gpus, config):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                        "--launch-check", "--config", config],
                       capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={k: v for k, v in os.environ.items()
                            if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_self_launches_ranks_and_shards():
    """`bench.py --gpus 2` without torchrun re-executes itself under
    torch.distributed.run (one rank per GPU; here gloo on CPU with
    --launch-check): both ranks come up, each takes its §8(e) KV-head block,
    the MAX over ranks reaches rank 0 and the head-major output gather is a
    plain concatenation."""
    d = _launch_check(2, "qwen3-32b_b64_ctx32k")
    assert d["n_gpus"] == 2 and d["gather_ok"] and d["max_over_ranks"] == 2.0
    assert d["shards_b0_bn_h0_hn"] == [[0, 64, 0, 4], [0, 64, 4, 4]]

