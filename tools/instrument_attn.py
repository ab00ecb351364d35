"""Apply (or check) the a5 timeline instrumentation patch to csrc/zoomr_attn.cu (debug only).
Usage: python tools/instrument_attn.py apply|revert"""
import os, sys, shutil
P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_10898_b200/csrc/zoomr_attn.cu")
BAK = "/tmp/zoomr_attn.cu.uninstrumented"
if sys.argv[1] == "revert":
    shutil.copy(BAK, P); sys.exit(0)
shutil.copy(P, BAK)
s = open(P).read()
rep = [
 ('struct TmaMaps {', '''__device__ unsigned long long g_tl[4][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL(who, k) if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77) && (warp % kPairs) == 0) g_tl[(blockIdx.x ? 2 : 0) + (who)][k] = gtime();

struct TmaMaps {'''),
 ('''  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Hq = p.Hkv * G;
''', '''  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Hq = p.Hkv * G;
  TL(warp >= kPairs ? 1 : 0, 0)
'''),
 ('''  asm volatile("griddepcontrol.wait;" ::: "memory");''', '''  asm volatile("griddepcontrol.wait;" ::: "memory");
  TL(warp >= kPairs ? 1 : 0, 1)'''),
 ('''  const int pair = warp % kPairs;
  const bool producer = warp >= kPairs;
  const int64_t gw =''', '''  const int pair = warp % kPairs;
  const bool producer = warp >= kPairs;
  TL(producer ? 1 : 0, 2)
  const int64_t gw ='''),
 ('''      if (lane == 0) mbar_arrive_expect_tx(&fullp[s], tx);''', '''      if (k == 0) TL(1, 3)
      if (lane == 0) mbar_arrive_expect_tx(&fullp[s], tx);'''),
 ('''      cp_async_arrive_noinc(&fullp[s]);
      q0 = q1;''', '''      cp_async_arrive_noinc(&fullp[s]);
      if (k == ntiles - 1) TL(1, 5)
      q0 = q1;'''),
 ('''    mbar_wait(&fullp[s], (uint32_t)((k / kStages) & 1));''', '''    if (k == 0) TL(0, 3)
    mbar_wait(&fullp[s], (uint32_t)((k / kStages) & 1));
    if (k == 0) TL(0, 4)'''),
 ('''  if (cur_b >= 0) flush(cur_b, cur_seg);
}''', '''  TL(0, 5)
  if (cur_b >= 0) flush(cur_b, cur_seg);
  TL(0, 6)
}'''),
]
for a, b in rep:
    assert a in s, a[:60]
    s = s.replace(a, b, 1)
s += '''
extern "C" int zoomr_debug_attn_timeline(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, zoomr::g_tl, sizeof(zoomr::g_tl)) == cudaSuccess ? 0 : 8;
}
'''
open(P, "w").write(s)
