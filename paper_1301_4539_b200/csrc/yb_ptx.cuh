// yb_ptx.cuh — sm_100a PTX helpers shared by the sweep kernels (mbarrier,
// TMA tensor loads, L2-hinted stores, warp shifts). Internal.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace yb {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "YB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra YB_WAIT;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// TMA prefetch of a box into L2 (no shared-memory destination, no barrier):
// raises the bytes in flight beyond what the shared-memory stage ring holds.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void sts4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ float& el(float4& v, int q) {
  return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}
__device__ __forceinline__ float elc(const float4& v, int q) {
  return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

// value at i-1 for each element of a lane's float4 (lane 0 reads `left`).
__device__ __forceinline__ float4 shift_im(float4 v, int lane, float left) {
  float w = __shfl_up_sync(0xffffffffu, v.w, 1);
  if (lane == 0) w = left;
  return make_float4(w, v.x, v.y, v.z);
}
// value at i+1 for each element (lane 31 reads `right`).
__device__ __forceinline__ float4 shift_ip(float4 v, int lane, float right) {
  float x = __shfl_down_sync(0xffffffffu, v.x, 1);
  if (lane == 31) x = right;
  return make_float4(v.y, v.z, v.w, x);
}

// 128-bit store with an L2 cache-policy hint (evict_first: the next-state
// arrays are not read again in this launch, so they should not push the
// halo rows neighbouring CTAs are about to read out of L2).
#ifndef YB_STG_MODE
#define YB_STG_MODE 0
#endif
__device__ __forceinline__ void stg4_hint(float* ptr, float4 v, uint64_t pol) {
#if YB_STG_MODE == 0
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
#elif YB_STG_MODE == 1
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol));
#elif YB_STG_MODE == 2
  (void)pol;
  __stcs(reinterpret_cast<float4*>(ptr), v);
#else
  (void)pol;
  *reinterpret_cast<float4*>(ptr) = v;
#endif
}

__device__ __forceinline__ void store_row4(float* base, long long p, int i0, int nx, float4 v,
                                           uint64_t pol) {
  if (i0 + 3 < nx) {
    stg4_hint(base + p, v, pol);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < nx) base[p + q] = elc(v, q);
  }
}

// the three components of one row behind a single ragged-edge branch
__device__ __forceinline__ void store_rows3(float* const* base, long long p, int i0, int nx, float4 v0,
                                            float4 v1, float4 v2, uint64_t pol) {
  float *b0 = base[0], *b1 = base[1], *b2 = base[2];
  if (i0 + 3 < nx) {
    stg4_hint(b0 + p, v0, pol);
    stg4_hint(b1 + p, v1, pol);
    stg4_hint(b2 + p, v2, pol);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < nx) {
        b0[p + q] = elc(v0, q);
        b1[p + q] = elc(v1, q);
        b2[p + q] = elc(v2, q);
      }
  }
}

}  // namespace
}  // namespace yb

namespace yb {
namespace {
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Device wall clock (ns) for the deadlines of the bounded spin waits.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A spin wait passed its deadline: the first one to time out fills the
// handle's wait-error record (WaitErr in yb_launch.h); the host reports it.
__device__ __forceinline__ void wait_timed_out(int* rec, int code, int item, int sweep, unsigned seen,
                                               unsigned need) {
  if (atomicCAS(rec, 0, -1) == 0) {
    rec[1] = item;
    rec[2] = sweep;
    rec[3] = (int)seen;
    rec[4] = (int)need;
    __threadfence();
    atomicExch(rec, code);
  }
}
}  // namespace
}  // namespace yb
