"""Debug: a5 early-known vs index-only on a config; where do outputs differ?"""
import os, sys, dataclasses, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zoomr_synth as S
from tests import parity as PY
cfg = dataclasses.replace(S.config_by_name(os.environ.get("WL", "8b32k")), batch=int(os.environ.get("B", "3")))
inp = S.generate(cfg, device="cuda")
a, b = PY.make_step(inp, capacity=8192), PY.make_step(inp, capacity=8192)
b.early_known = False
PY.run_full(inp, a, fused=True)
PY.run_full(inp, b, fused=True)
print("count", a.count.tolist(), "seq_len", inp.seq_len.tolist())
d = (a.out - b.out).abs().amax(dim=-1)  # [B][L][Hq]
print("max diff", d.max().item())
bad = (d > 1e-5).nonzero().tolist()
print("n bad (b,l,h)", len(bad), bad[:20])
G = cfg.Hq // cfg.Hkv
segs = sorted({(x[0], x[1] * cfg.Hkv + x[2] // G) for x in bad})
print("bad segments (b, l*Hkv+g)", len(segs), segs[:40])
