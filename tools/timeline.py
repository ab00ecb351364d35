"""Step timeline from the ZOOMR_TIMELINE experiment build (globaltimer marks, min/max over the grid).

  python -c "from paper_2604_10898_b200 import _build; _build.build(out='ablibs/lib_tl.so', defines=['ZOOMR_TIMELINE'])"
  ZOOMR_LIB_OVERRIDE=$PWD/ablibs/lib_tl.so python tools/timeline.py      (VARS=early,late WL=8b16k)
Marks (us after the first select CTA started), each as min..max over CTAs / warps:
  select: 0 CTA start, 1 front end (before ticket), 2 tail start, 3 collected, 4 top-c done, 5 last CTA end
  a5:     0 CTA start, 1 prologue done, 2 phase-B schedule known, 3 first tile landed, 4 first B tile landed,
          5 math warp done, 6 producer done"""
import ctypes as C, os, sys, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from paper_2604_10898_b200 import zoomr as Z
from paper_2604_10898_b200.step import StepParams, ZoomrStep

cfg = S.config_by_name(os.environ.get("WL", "8b16k"))
if os.environ.get("HKV"):  # a head shard's geometry (e.g. HKV=1 HQ=8 for one rank of 70B-64K over 8)
    import dataclasses
    cfg = dataclasses.replace(cfg, Hkv=int(os.environ["HKV"]), Hq=int(os.environ["HQ"]))
shape = Z.Shape(cfg.L, cfg.Hq, cfg.Hkv, cfg.d, cfg.page)
lib = Z.lib()
for fn in ("zoomr_tl_arm_fused", "zoomr_tl_arm_attn"):
    getattr(lib, fn).argtypes = [C.c_int, C.c_void_p]
U64 = C.c_ulonglong * 32


def read(fn, reset):
    b = U64()
    assert fn(b, reset) == 0
    return list(b)


NAMES = {"select": ["start", "front_end", "tail_start", "collected", "topc_done", "end", "a1_done", "(unused)",
                    "score_topk_done", "score_loop_done(warp)", "score_loop_start"],
         "a5": ["start", "prologue", "B_known", "first_tile", "first_B_tile", "math_done", "prod_done",
                "first_issue", "prod_enter", "first_stage_a"]}
for var in os.environ.get("VARS", "early,late").split(","):
    sets = []
    for r in range(4):
        inp = S.generate(cfg, device="cuda", seed=cfg.seed + 17 * r)
        st = ZoomrStep(shape, 1, inp.bounds.shape[1], cfg.T, StepParams(cfg.top_k, cfg.c, cfg.sink, cfg.window),
                       early_known=(var == "early"))
        kv = (inp.k_pool, inp.v_pool, inp.page_table); seg = (inp.bounds, inp.num_summaries, inp.seq_len)
        st.update_mean_keys(kv, seg, st.all_items(inp.num_summaries))
        newest = torch.tensor([[0, int(inp.num_summaries[0]) - 1]], dtype=torch.int32, device="cuda")
        g = st.capture(inp.q, kv, seg, close_items=newest)
        if os.environ.get("A5ONLY"):  # a graph of a5 alone (over the I_f the step above left)
            st.run(inp.q, kv, seg, close_items=newest)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                st.attend(inp.q, kv, inp.seq_len if var == "early" else None)
        g.keep = (st, inp, newest)  # the graph uses their buffers
        sets.append(g)
    for i in range(12):
        sets[i % 4].replay()
    torch.cuda.synchronize()
    samples = []
    def measured_step(i):
        """Warm steps back to back, then the marked step (armed in stream order): clocks stay up."""
        read(lib.zoomr_tl_fused, 1); read(lib.zoomr_tl_attn, 1)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for a in (lib.zoomr_tl_arm_fused, lib.zoomr_tl_arm_attn):
            a(0, st)
        for j in range(8):
            sets[(i + j) % 4].replay()
        for a in (lib.zoomr_tl_arm_fused, lib.zoomr_tl_arm_attn):
            a(1, st)
        sets[i % 4].replay()
        for a in (lib.zoomr_tl_arm_fused, lib.zoomr_tl_arm_attn):
            a(0, st)
        torch.cuda.synchronize()

    for i in range(int(os.environ.get("REPS", "8"))):
        measured_step(i)
        samples.append((read(lib.zoomr_tl_fused, 0), read(lib.zoomr_tl_attn, 0)))
    print(f"== {var} ({cfg.name}), median over {len(samples)} steps, us after the first select CTA start")
    for who, idx in (("select", 0), ("a5", 1)):
        for m, name in enumerate(NAMES[who]):
            base = lambda s: s[0][0] if s[0][0] != 2**64 - 1 else s[1][0]  # A5ONLY: the first a5 CTA start
            lo = [s[idx][2 * m] - base(s) for s in samples if s[idx][2 * m] != 2**64 - 1]
            hi = [s[idx][2 * m + 1] - base(s) for s in samples if s[idx][2 * m + 1]]
            if lo:
                print(f"  {who:6s} {m} {name:12s} {statistics.median(lo)/1e3:8.2f} .. {statistics.median(hi)/1e3:8.2f}")

# per-CTA end times vs SM id (is the a5 tail imbalance systematic?)
if os.environ.get("CTA"):
    import collections
    ends = collections.defaultdict(list)
    starts = collections.defaultdict(list)
    for i in range(int(os.environ.get("REPS", "8"))):
        measured_step(i)
        f = read(lib.zoomr_tl_fused, 0)
        buf = (C.c_ulonglong * 4096)()
        lib.zoomr_tl_cta_attn(buf)
        for c in range(148):
            smid, t0, t1 = buf[4 * c], buf[4 * c + 1], buf[4 * c + 2]
            if t1:
                ends[smid].append((t1 - f[0]) / 1e3)
                starts[smid].append((t0 - f[0]) / 1e3)
    rows = sorted((statistics.median(v), sm, statistics.median(starts[sm]), min(v), max(v)) for sm, v in ends.items())
    print("a5 CTA end (median over reps), by SM: fastest 10 / slowest 10   [sm, start, end min..max]")
    for r in rows[:10] + rows[-10:]:
        print(f"  sm {r[1]:3d} start {r[2]:6.2f} end {r[0]:6.2f} ({r[3]:6.2f}..{r[4]:6.2f})")
    # rank correlation between two halves of the reps
    a = {sm: statistics.median(v[: len(v) // 2]) for sm, v in ends.items()}
    b = {sm: statistics.median(v[len(v) // 2:]) for sm, v in ends.items()}
    sms = sorted(a)
    ra = {sm: i for i, sm in enumerate(sorted(sms, key=lambda s: a[s]))}
    rb = {sm: i for i, sm in enumerate(sorted(sms, key=lambda s: b[s]))}
    n = len(sms)
    rho = 1 - 6 * sum((ra[s] - rb[s]) ** 2 for s in sms) / (n * (n * n - 1))
    print("spearman(first half, second half) =", round(rho, 3))
    # by SM pairs (TPC) and by sm // 16 groups
    grp = collections.defaultdict(list)
    for sm, v in ends.items():
        grp[sm // 18].append(statistics.median(v))
    print("median end by smid//18:", {k: round(statistics.median(v), 2) for k, v in sorted(grp.items())})

# per-math-warp counters: end time vs tiles / merges / cp.async rows / boxes
if os.environ.get("WARPS"):
    recs = []
    for i in range(int(os.environ.get("REPS", "8"))):
        measured_step(i)
        f = read(lib.zoomr_tl_fused, 0)
        buf = (C.c_ulonglong * (4096 * 8))()
        lib.zoomr_tl_warp_attn(buf)
        for w in range(4096):
            r = buf[8 * w: 8 * w + 8]
            if r[0]:
                recs.append(dict(rep=i, w=w, end=(r[0] - f[0]) / 1e3, tiles=r[1], merges=r[2], merge_us=r[3] / 1e3,
                                 cp_rows=r[4], boxes=r[5], pend=(r[6] - f[0]) / 1e3 if r[6] else 0, flushes=r[7]))
    import json, numpy as np
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(recs, open("gpurun_out/timeline_warps.json", "w"))
    keys = ["end", "tiles", "merges", "merge_us", "cp_rows", "boxes", "pend", "flushes"]
    M = np.array([[r[k] for k in keys] for r in recs], dtype=np.float64)
    print("per-warp stats over", len(recs), "warp-steps")
    for j, k in enumerate(keys):
        print(f"  {k:9s} mean {M[:, j].mean():9.2f} min {M[:, j].min():9.2f} max {M[:, j].max():9.2f}")
    for j, k in enumerate(keys[1:], 1):
        print(f"  corr(end, {k:9s}) = {np.corrcoef(M[:, 0], M[:, j])[0, 1]:+.3f}")
    # end time of warp w within its CTA: by pair index
    for pidx in range(4):
        sel = M[[r["w"] % 4 == pidx for r in recs]]
        print(f"  pair {pidx}: mean end {sel[:, 0].mean():.2f}")
    # linear fit end ~ a + b*cp_rows + c*boxes + d*merge_us
    X = np.c_[np.ones(len(M)), M[:, 4], M[:, 5], M[:, 3], M[:, 7]]
    coef, *_ = np.linalg.lstsq(X, M[:, 0], rcond=None)
    print("  fit end = %.2f + %.4f*cp_rows + %.4f*boxes + %.3f*merge_us + %.3f*flushes" % tuple(coef))

# producer ramp in SM clocks (the ZOOMR_TL_RAMP build: fields 4 / 5 / 3 / 7 hold clock64 at
# producer entry, after its first stage_a, at its first copy issue, and at its math warp's first tile)
if os.environ.get("RAMP"):
    import numpy as np
    d1, d2, d3 = [], [], []
    for i in range(int(os.environ.get("REPS", "8"))):
        measured_step(i)
        buf = (C.c_ulonglong * (4096 * 8))()
        lib.zoomr_tl_warp_attn(buf)
        for w in range(4096):
            r = buf[8 * w: 8 * w + 8]
            if r[4] and r[5] and r[3] and r[7]:
                d1.append(r[5] - r[4]); d2.append(r[3] - r[5]); d3.append(r[7] - r[3])
    for name, v in (("enter -> first stage_a", d1), ("first stage_a -> first issue", d2),
                    ("first issue -> math warp's first tile", d3)):
        v = np.array(v, dtype=np.float64)
        print(f"  {name:40s} cycles p10 {np.percentile(v, 10):8.0f} p50 {np.median(v):8.0f} p90 {np.percentile(v, 90):8.0f}")
