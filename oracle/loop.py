"""Algorithm 1's decode loop over the oracle (TEST INFRASTRUCTURE ONLY, see
``oracle/__init__.py``): the reference for the device loop
(zoomr_append_kv + zoomr_track_segments + zoomr_select_fused with update flags
+ zoomr_sparse_decode_attn).

Per step, in Algorithm 1's order:
  1. append k_t, v_t (Alg.1 @P:407) -- T += 1;
  2. segment tracking (SPEC ingest_token S:36-45): begin delimiter at position j
     freezes the open tail [tail, j) as the pending R and opens a summary at j;
     end delimiter at j closes S = [open, j + 1) (delimiters included), appends
     (R, S) and computes the new summary's mean keys (Alg.1 @P:408-409, O1);
  3. at a semantic-boundary token (the preset list) the selection is
     updated with q_t: scores, per-head top-k, votes, consensus (O2-O5 over all
     closed summaries); otherwise the flags from the last update are kept
     (reading Q14; summaries closed since then have flag 0);
  4. I_f from the current segments, flags and T (O6), attention (O7).
The arithmetic is the oracle's C functions; this file only sequences them."""
from __future__ import annotations

import numpy as np

from . import oracle as O


class OracleLoop:
    def __init__(self, L, Hq, Hkv, d, top_k, c, sink, window, begin_id, end_id, boundary_ids,
                 prompt_k, prompt_v):
        self.L, self.Hq, self.Hkv, self.d = L, Hq, Hkv, d
        self.top_k, self.c, self.sink, self.window = top_k, c, sink, window
        self.begin_id, self.end_id, self.boundary = begin_id, end_id, set(int(x) for x in boundary_ids)
        self.K = [np.asarray(r, dtype=np.uint16) for r in prompt_k]  # rows [L][Hkv][d] bf16 bits
        self.V = [np.asarray(r, dtype=np.uint16) for r in prompt_v]
        n_p = len(self.K)
        self.open, self.tail, self.pend = -1, n_p, (n_p, n_p)
        self.segs = []          # (r0, r1, s0, s1)
        self.mk = []            # per summary: double [L][Hkv][d]
        self.flags = np.zeros(0, np.uint8)
        self.last = {}

    @property
    def T(self):
        return len(self.K)

    def step(self, k_new, v_new, q, token_id):
        self.K.append(np.asarray(k_new, dtype=np.uint16))
        self.V.append(np.asarray(v_new, dtype=np.uint16))
        pos = self.T - 1
        closed = -1
        if token_id == self.begin_id:
            if self.open >= 0:
                raise ValueError("NestedSummary")
            self.pend = (self.tail, pos)
            self.open = pos
        elif token_id == self.end_id:
            if self.open < 0:
                raise ValueError("UnmatchedEnd")
            seg = (self.pend[0], self.pend[1], self.open, pos + 1)
            self.segs.append(seg)
            keys = np.stack(self.K)
            self.mk.append(O.update_mean_keys(keys, np.array([seg], np.int32), self.L, self.Hkv, self.d)[:, :, 0])
            closed = len(self.segs) - 1
            self.open, self.tail = -1, pos + 1
        n = len(self.segs)
        flags = np.zeros(n, np.uint8)
        flags[: len(self.flags)] = self.flags[:n]
        update = int(token_id) in self.boundary
        votes = A = None
        if update:
            if n:
                mk = np.stack(self.mk, axis=2)  # [L][Hkv][n][d]
                sc = O.score(q, mk, self.top_k, self.L, self.Hq, self.Hkv, self.d)
                votes, A = sc["votes"], sc["A"]
                flags = O.select_topc(votes, A, self.c)[0]
            else:
                flags = np.zeros(0, np.uint8)
        self.flags = flags
        seg_arr = np.array(self.segs, np.int32).reshape(-1, 4)
        idx = O.build_index(seg_arr, flags, self.T, self.sink, self.window)
        out = O.sparse_decode_attn(q, np.stack(self.K), np.stack(self.V), idx, self.L, self.Hq, self.Hkv, self.d)
        self.last = dict(closed=closed, update=update, flags=flags.copy(), index=idx, out=out, votes=votes, A=A,
                         segs=seg_arr.copy())
        return self.last
