"""Wait-time budget of the decode kernel (instrumented build), config [2]."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ASYNCSPADE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_32B, "cuda")
step.fill_synthetic()
step.run()
torch.cuda.synchronize()
L = asp.lib()
buf = (ctypes.c_ulonglong * 16)()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    L.asp_decode_prof_read(buf)
    ev[0].record()
    asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx, out=step.out, workspace=step.ws_dec, params=step.p_dec)
    ev[1].record()
    torch.cuda.synchronize()
L.asp_decode_prof_read(buf)
print("decode call us", ev[0].elapsed_time(ev[1]) * 1000)
names = ["P qempty", "P tokempty", "P stage-empty", "M stage-full", "M qfull", "M pfull", "M oempty",
         "S tokfull", "S sfull", "E ofull", "cta total", "P cp.async wait"]
for n, v in zip(names, buf):
    print(f"{n:14s} {v / 148 / 1.93e3:8.1f} us/CTA")
