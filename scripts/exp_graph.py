"""Eager vs CUDA-graph replay of the config [2] step (device events around K steps)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
P = int(os.environ.get("SHARD", "1"))
step = DecodeStep(configs.QWEN3_32B, "cuda", kv_heads=(0, 8 // P))
step.fill_synthetic()
K = 20
def timeit(f):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
print("eager us/step", timeit(step.run))
step.capture()
print("graph us/step", timeit(step.replay))
print("eager us/step", timeit(step.run))
