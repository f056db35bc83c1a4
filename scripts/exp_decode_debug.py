"""Cold-L2 decode with the S-recompute check (debug build)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ASYNCSPADE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_8B, "cuda")
step.fill_synthetic()
step.run(); torch.cuda.synchronize()
L = asp.lib()
buf = (ctypes.c_ulonglong * 16)()
junk = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for it in range(3):
    junk.fill_(it); torch.cuda.synchronize()
    L.asp_decode_prof_read(buf)
    asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx, out=step.out, workspace=step.ws_dec, params=step.p_dec)
    torch.cuda.synchronize()
    L.asp_decode_prof_read(buf)
    print("cold run", it, "S mismatches", buf[12], "of", buf[13], "V chunk mismatches", buf[14], "tiles", buf[15])
