"""Summarise tools/ab_probe.sh output (records span two lines: the probe's JSON ends with a newline)."""
import json
import sys

txt = open(sys.argv[1]).read()
dec = json.JSONDecoder()
i = 0
rows = []
while True:
    j = txt.find("{", i)
    if j < 0:
        break
    try:
        d, end = dec.raw_decode(txt, j)
    except json.JSONDecodeError:
        i = j + 1
        continue
    rows.append(d)
    i = end
for d in rows:
    p = d.get("probe")
    if not p:
        print(d.get("lib"), "failed")
        continue
    print(f"{d['lib']:22s} r{d['round']} {p['cfg']:10s} Hkv={p['Hkv']} a5_idx {p['a5_index_only_us']:6.1f} "
          f"a5_early {p['a5_early_us']:6.1f} sel {p['select_fused_us']:5.1f} step {p['step_fused_us']:6.1f} "
          f"single {p.get('step_single_replay_us', 0):6.1f} sep {p['step_separate_us']:6.1f} held {p['step_held_us']:6.1f} | frac {p['a5_index_only_frac']:.3f} "
          f"{p['a5_early_frac']:.3f}")
