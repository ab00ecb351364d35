// common.cuh -- shared device/host helpers of libzoomr (sm_100a).
// Product code: never includes or links anything under oracle/.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/zoomr.h"

namespace zoomr {

constexpr int kMaxSummaries = 4096;  // N_max supported by a2/a3/a4 (shared-memory resident)
constexpr int kMaxTopK = 32;

// First device-detected error wins (zoomr.h "Errors").
__device__ __forceinline__ void set_status(int32_t *st, int32_t code) {
  if (st) atomicCAS(st, 0, code);
}

__device__ __forceinline__ float bf16lo_to_float(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi_to_float(uint32_t w) {
  return __uint_as_float(w & 0xffff0000u);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The library's only host state: per stream, the kind of its own most recent
// launch (and the a5 workspace it used).  It lets a call detect, at enqueue
// time, the one launch order whose overlap would be unsafe -- a PDL-launched
// a5 that writes its workspace before griddepcontrol.wait, enqueued right
// behind a chained a5 on the same workspace -- and fall back to the
// serialised variant instead of racing (zoomr.h "Chained launches").  Stream
// order is enqueue order, also under graph capture, so the record is exact for
// the library's own launches; a foreign kernel in between only makes the
// fallback conservative.  A stale entry (a destroyed stream whose handle is
// reused) can likewise only cause a conservative fallback.
enum LaunchKind : int { kLaunchOther = 0, kLaunchA5Chained = 1 };
void note_launch(cudaStream_t s, int kind, const void *ws);
bool prev_launch_is(cudaStream_t s, int kind, const void *ws);  // ws == nullptr: any workspace

inline int launch_status(cudaStream_t s, int kind = kLaunchOther, const void *ws = nullptr) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ZOOMR_ERR_CUDA;
  note_launch(s, kind, ws);
  return ZOOMR_OK;
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  }
  return n;
}

// Every libzoomr kernel asks for the maximum shared-memory carveout so that
// consecutive kernels of a step never force an L1/shared re-partition of the
// SMs (env ZOOMR_CARVEOUT=-1 disables, for A/B measurements).
template <typename F>
inline void prefer_max_smem(F *kfn) {
  static int mode = -2;
  if (mode == -2) {
    const char *e = getenv("ZOOMR_CARVEOUT");
    mode = e ? atoi(e) : -1;  // default: leave the carveout to the driver (measured best)
  }
  if (mode >= 0) cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, mode);
}

// Launch with programmatic dependent launch (PDL): the kernel may start while
// its predecessor on the stream is finishing; it must execute
// `griddepcontrol.wait` before touching the predecessor's outputs.
template <typename Kern, typename... Args>
inline void launch_pdl(Kern kfn, dim3 grid, int block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static int no_pdl = -1;
  if (no_pdl < 0) {
    const char *e = getenv("ZOOMR_NO_PDL");  // A/B experiments only
    no_pdl = e ? atoi(e) : 0;
  }
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kfn, args...);
}

// Cooperative launch: the whole grid is co-resident (the launch fails if it
// cannot be), which kernels whose CTAs wait on one another require.
template <typename Kern, typename... Args>
inline void launch_cooperative(Kern kfn, dim3 grid, int block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kfn, args...);
}

// Let the next kernel on the stream (launched with PDL) begin its prologue.
__device__ __forceinline__ void allow_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool valid_geom(const zoomr_geom *g) {
  if (!g) return false;
  if (g->num_layers < 1 || g->num_q_heads < 1 || g->num_kv_heads < 1 || g->page_size < 1) return false;
  return true;
}

inline int check_geom(const zoomr_geom *g) {
  if (!valid_geom(g)) return ZOOMR_ERR_INVALID_ARG;
  if (g->num_q_heads % g->num_kv_heads) return ZOOMR_ERR_DIM_MISMATCH;
  int G = g->num_q_heads / g->num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 7 && G != 8) return ZOOMR_ERR_DIM_MISMATCH;  // 7: Qwen2.5-7B (28 / 4)
  int d = g->head_dim;
  if (d != 16 && d != 32 && d != 64 && d != 128) return ZOOMR_ERR_UNSUPPORTED;
  return ZOOMR_OK;
}

}  // namespace zoomr

// ---- experiment builds only (-DZOOMR_TIMELINE, tools/timeline.py) ----------
// TL(i): lane 0 records %globaltimer into the min / max of slot i of the
// translation unit's g_tl (declare with ZOOMR_TL_STORAGE(name), which also
// exports zoomr_tl_<name>(out, reset)).  Compiled out of the product library.
#ifdef ZOOMR_TIMELINE
#define ZOOMR_TL_STORAGE(name)                                                                    \
  namespace zoomr {                                                                               \
  static __device__ unsigned long long g_tl[2 * 16];                                              \
  static __device__ int g_tl_on; /* marks are recorded only while armed */                        \
  }                                                                                               \
  extern "C" int zoomr_tl_arm_##name(int on, void *stream) {                                      \
    static int v[2] = {0, 1};                                                                     \
    return cudaMemcpyToSymbolAsync(zoomr::g_tl_on, &v[on ? 1 : 0], sizeof(int), 0,                \
                                   cudaMemcpyHostToDevice, (cudaStream_t)stream) == cudaSuccess ? 0 : 8; \
  }                                                                                               \
  ZOOMR_TL_STORAGE_REST(name)
#define ZOOMR_TL_STORAGE_REST(name)                                                               \
  namespace zoomr {                                                                               \
  static __device__ unsigned long long g_tl_cta[1024][4]; /* per CTA: smid, start, end, - */       \
  static __device__ unsigned long long g_tl_warp[4096][8]; /* per math warp: free-form counters */  \
  }                                                                                               \
  extern "C" int zoomr_tl_warp_##name(unsigned long long *out) {                                  \
    return cudaMemcpyFromSymbol(out, zoomr::g_tl_warp, sizeof(zoomr::g_tl_warp)) == cudaSuccess ? 0 : 8; \
  }                                                                                               \
  extern "C" int zoomr_tl_cta_##name(unsigned long long *out) {                                   \
    return cudaMemcpyFromSymbol(out, zoomr::g_tl_cta, sizeof(zoomr::g_tl_cta)) == cudaSuccess ? 0 : 8; \
  }                                                                                               \
  extern "C" int zoomr_tl_##name(unsigned long long *out, int reset) {                            \
    if (cudaMemcpyFromSymbol(out, zoomr::g_tl, sizeof(zoomr::g_tl)) != cudaSuccess) return 8;    \
    if (reset) {                                                                                  \
      unsigned long long h[2 * 16];                                                               \
      for (int i = 0; i < 16; ++i) { h[2 * i] = ~0ull; h[2 * i + 1] = 0; }                        \
      if (cudaMemcpyToSymbol(zoomr::g_tl, h, sizeof(h)) != cudaSuccess) return 8;                \
      void *pc = nullptr;                                                                         \
      if (cudaGetSymbolAddress(&pc, zoomr::g_tl_cta) != cudaSuccess) return 8;                    \
      if (cudaMemset(pc, 0, sizeof(zoomr::g_tl_cta)) != cudaSuccess) return 8;                    \
      if (cudaGetSymbolAddress(&pc, zoomr::g_tl_warp) != cudaSuccess) return 8;                   \
      if (cudaMemset(pc, 0, sizeof(zoomr::g_tl_warp)) != cudaSuccess) return 8;                   \
    }                                                                                             \
    return 0;                                                                                     \
  }
#define TL(i)                                                                  \
  do {                                                                         \
    if ((threadIdx.x & 31) == 0 && tl_on_) {                \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      atomicMin(&g_tl[2 * (i)], t_);                                           \
      atomicMax(&g_tl[2 * (i) + 1], t_);                                       \
    }                                                                          \
  } while (0)
// TL_CTA(k): per-CTA record (k = 1 start, 2 end: max over the CTA's warps), slot 0 = %smid
#define TL_CTA(k)                                                                          \
  do {                                                                                     \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024 && tl_on_) {       \
      unsigned long long t_;                                                               \
      unsigned sm_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                     \
      g_tl_cta[blockIdx.x][0] = sm_;                                                       \
      if ((k) == 1) g_tl_cta[blockIdx.x][1] = t_;                                          \
      else atomicMax(&g_tl_cta[blockIdx.x][k], t_);                                        \
    }                                                                                      \
  } while (0)
#define TL_INIT() const bool tl_on_ = *(volatile int *)&g_tl_on  // once per kernel: marks only while armed
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t_;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
  return t_;
}
#define TLW_ADD(w, f, v) do { if ((threadIdx.x & 31) == 0 && (w) < 4096 && tl_on_) atomicAdd(&g_tl_warp[w][f], (unsigned long long)(v)); } while (0)
#define TLW_SET(w, f, v) do { if ((threadIdx.x & 31) == 0 && (w) < 4096 && tl_on_) g_tl_warp[w][f] = (unsigned long long)(v); } while (0)
#define TL_NOW() tl_now()
#else
#define ZOOMR_TL_STORAGE(name)
#define TL(i) do { } while (0)
#define TL_CTA(k) do { } while (0)
#define TLW_ADD(w, f, v) do { } while (0)
#define TLW_SET(w, f, v) do { } while (0)
#define TL_NOW() 0ull
#define TL_INIT() do { } while (0)
#endif
