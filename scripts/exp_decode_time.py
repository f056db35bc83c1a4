"""Time sparse_decode alone at config [2] for the library in ASYNCSPADE_LIB."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_32B, "cuda")
step.fill_synthetic(); step.run(); torch.cuda.synchronize()
junk = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for it in range(6):
    junk.fill_(it)
    ev[0].record()
    asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx, out=step.out, workspace=step.ws_dec, params=step.p_dec)
    ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1000)
print(os.path.basename(os.environ.get("ASYNCSPADE_LIB", "default")), "decode us (cold L2):", sorted(ts)[len(ts)//2])
