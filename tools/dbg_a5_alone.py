"""a5 launched alone (no preceding select kernel) in early-known mode: must match index-only."""
import os, sys, dataclasses, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from tests import parity as PY
name = os.environ.get("WL", "tiny")
cfg = S.config_by_name(name)
if os.environ.get("B"):
    cfg = dataclasses.replace(cfg, batch=int(os.environ["B"]))
inp = S.generate(cfg, device="cuda", seed=3)
st = PY.make_step(inp, capacity=8192 if name != "tiny" else None)
st.early_known = False
PY.run_full(inp, st, fused=True)
ref = st.out.clone()
kv = (inp.k_pool, inp.v_pool, inp.page_table)
for mode in (False, True, True, False, True):
    st.early_known = mode
    st.out.zero_()
    st.attend(inp.q, kv, inp.seq_len)
    torch.cuda.synchronize()
    print(name, "early" if mode else "index", "max diff", (st.out - ref).abs().max().item(), flush=True)

# back-to-back launches inside one graph (PDL edges between consecutive a5 nodes)
if os.environ.get("GRAPH"):
    for mode in (False, True):
        st.early_known = mode
        sep = os.environ.get("SEP") == "1"
        dummy = torch.zeros(1, device="cuda")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                st.attend(inp.q, kv, inp.seq_len)
                if sep:
                    dummy.add_(1.0)
        g.replay()
        torch.cuda.synchronize()
        print("graph", "early" if mode else "index", "sep" if sep else "", "max diff", (st.out - ref).abs().max().item(), flush=True)
