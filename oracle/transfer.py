"""SPEC's transfer-schedule model of the paper's layer-pipelined host tier
(TEST INFRASTRUCTURE ONLY, see ``oracle/__init__.py``).

PAPER.md P:109 (section 3.4, "System Implementation and Inference"): "For each
layer of the model, the required KV cache slices are transferred to the GPU.
Once the layer's computation is finished, its KVs are asynchronously
transferred back to the CPU while the KVs for the next layer are prefetched."
SPEC.md S:286-294 `simulate_transfer_schedule` states it as a two-stage
pipeline: layer l's compute overlaps layer l+1's transfer-in and layer l-1's
transfer-out; at most two slices are resident (current + prefetched);
total_time = when the last layer's compute and write-back complete under the
greedy schedule; serial_time = sum of transfer-in + compute + transfer-out.

Discrete-event reading (S:291's hand simulation: in [2,2,2], compute [3,3,3],
free write-back -> 2 + 3*3 = 11 vs serial 15):
  * one inbound engine and one outbound engine (a duplex host link), each
    serving its transfers in layer order;
  * in(l) starts when in(l-1) has finished and a slice slot is free: slot of
    layer l is freed when layer l-2's write-back has finished (two slots);
  * compute(l) starts when in(l) and compute(l-1) have finished;
  * out(l) starts when compute(l) and out(l-1) have finished.
Pure Python, every quantity a plain float."""
from __future__ import annotations


def simulate_transfer_schedule(t_in, t_compute, t_out=None, slots: int = 2):
    """Returns dict(total_time, serial_time, peak_resident_layers, events=[(l, in0, in1, c0, c1, o0, o1)])."""
    n = len(t_in)
    if len(t_compute) != n:
        raise ValueError("one compute time per layer")
    t_out = [0.0] * n if t_out is None else list(t_out)
    if len(t_out) != n or slots < 1:
        raise ValueError("bad transfer model")
    in_end, c_end, o_end = [0.0] * n, [0.0] * n, [0.0] * n
    events = []
    for l in range(n):
        slot_free = o_end[l - slots] if l >= slots else 0.0
        in0 = max(in_end[l - 1] if l else 0.0, slot_free)
        in_end[l] = in0 + t_in[l]
        c0 = max(in_end[l], c_end[l - 1] if l else 0.0)
        c_end[l] = c0 + t_compute[l]
        o0 = max(c_end[l], o_end[l - 1] if l else 0.0)
        o_end[l] = o0 + t_out[l]
        events.append((l, in0, in_end[l], c0, c_end[l], o0, o_end[l]))
    # resident slices: a layer's slice lives from the start of its transfer-in to the end of its write-back
    peak = 0
    for (_, a, _, _, _, _, _) in events:
        live = sum(1 for (_, a2, _, _, _, _, e2) in events if a2 <= a < e2)
        peak = max(peak, live)
    total = max(max(c_end), max(o_end)) if n else 0.0
    serial = sum(t_in) + sum(t_compute) + sum(t_out)
    return {"total_time": total, "serial_time": serial, "peak_resident_layers": peak, "events": events}
