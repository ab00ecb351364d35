"""A/B of a5 alone across library builds on the same box (any ABI version).

usage: python tools/ab_a5.py lib1.so lib2.so ...   (WL=8b16k, ROUNDS=2)
The index sets come from the current build's step (fused select); each listed
library's zoomr_sparse_decode_attn is then timed on them (graph of 20 launches,
4 rotating input sets), index-only mode and, for ABI >= 2, early-known mode."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep

cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
sets = []
for r in range(4):
    inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
    st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window))
    kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
    st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
    st.run(inp.q, kv, seg)
    sets.append((inp, st))
torch.cuda.synchronize()
vp, i32, sz = C.c_void_p, C.c_int32, C.c_size_t


def timer(lib, early):
    L = C.CDLL(os.path.abspath(lib))
    ver = L.zoomr_abi_version()
    if early and ver < 2:
        return None
    L.zoomr_attn_workspace_bytes.argtypes = [vp, i32]
    L.zoomr_attn_workspace_bytes.restype = sz
    g = shape.c()
    graphs = []
    for inp, st in sets:
        wsb = L.zoomr_attn_workspace_bytes(C.byref(g), 1)
        ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
        out = torch.empty_like(st.out)
        kv = Z._kv(inp.k_pool, inp.v_pool, inp.page_table)
        p = lambda t: C.c_void_p(t.data_ptr())
        if ver >= 2:
            L.zoomr_sparse_decode_attn.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, vp, i32, i32, C.c_float, vp, vp,
                                                   sz, vp, vp]
            args = lambda: (C.byref(g), 1, p(inp.q), C.byref(kv), p(st.index), None, p(st.count), st.index.shape[1],
                            p(inp.seq_len) if early else None, cfg.sink, cfg.window, C.c_float(cfg.d ** -0.5),
                            p(out), p(ws), wsb, None, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        else:
            L.zoomr_sparse_decode_attn.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32, C.c_float, vp, vp, sz, vp, vp]
            args = lambda: (C.byref(g), 1, p(inp.q), C.byref(kv), p(st.index), None, p(st.count), st.index.shape[1],
                            C.c_float(cfg.d ** -0.5), p(out), p(ws), wsb, None,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert L.zoomr_sparse_decode_attn(*args()) == 0
        torch.cuda.synchronize()
        assert (out - st.out).abs().max().item() < 1e-4, "output differs"
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    L.zoomr_sparse_decode_attn(*args())
        graphs.append((gr, ws, out))
    def run(K=40):
        for i in range(8): graphs[i % 4][0].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(K): graphs[i % 4][0].replay()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (K * 20)
    return run


runs = []
for lib in sys.argv[1:]:
    for early in (False, True):
        t = timer(lib, early)
        if t: runs.append((f"{lib} {'early' if early else 'index-only'}", t))
for r in range(int(os.environ.get("ROUNDS", "2"))):
    for name, f in runs:
        print(f"{name}: {f():.2f} us/launch", flush=True)
