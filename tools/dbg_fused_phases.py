import ctypes as C, torch, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import zoomr_synth as S
from tests import parity as PY
from paper_2604_10898_b200 import zoomr as Z
inp = S.generate(S.CONFIGS["8b16k"], device="cuda")
st = PY.make_step(inp, debug=False)
PY.run_full(inp, st, fused=True)
kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
lib = Z.lib()
for rep in range(5):
    torch.cuda.synchronize()
    Z.select_fused(st.shape, inp.q, inp.k_pool, inp.v_pool, inp.page_table, inp.bounds, inp.num_summaries, inp.seq_len,
                   newest, st.mean_keys, 2, 4, 4, 512, st.flags, st.index, st.count, st.sel_workspace, partial=st.partial,
                   index_phys=None)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 32)()
    lib.zoomr_debug_timestamps(buf)
    t = list(buf)
    base = min(x for x in t if x)
    print("last:", [round((x - base)/1000, 2) if x else None for x in t[16:32]])
