// yb_fused.cu — the FUSED one-sweep Yee step for sm_100a.
//
// One CTA owns a kTX x kTY column of cells (x,y) and marches a z-chunk of
// planes. Per plane k it
//   1. waits for the TMA-staged plane k of all read arrays (ex..hz of the
//      current state + the per-cell coefficient arrays), box x0-4..x0+TX+3,
//      y0-1..y0+TY, landed in a ring of `nstages` shared-memory stages by
//      cp.async.bulk.tensor + mbarrier complete_tx;
//   2. computes E^{n+1} on plane k for the owned cells plus the +x column and
//      +y row halo (update_e_dof, kernels.hpp:27-44, PEC folded in as "not
//      curl-updatable -> +0", staggering.hpp:70-86, sources added after it,
//      schedule.hpp:175-199), keeps it in a 3-deep shared plane buffer and
//      writes the owned part to the next state;
//   3. computes H^{n+3/2} on plane k-1 (update_h_dof, kernels.hpp:46-63) from
//      E^{n+1} planes k-1 (with halo) and k (own, registers) and the H / Da /
//      Db values of plane k-1 the same threads read one iteration earlier.
// This is planeAmpere(k); planeFaraday(k-1) of the paper's one-sweep scheme
// with the +x/+y E halo recomputed instead of exchanged.
// State is double-buffered (read `in`, write `out`), so CTAs never race on
// halo values; DRAM traffic is one read + one write of each field plus one
// read of each per-cell coefficient array per step.
// Arithmetic: yee_upd (explicit _rn intrinsics), bit-identical to the oracle.
#include <cuda.h>
#include <cuda_runtime.h>

#include "yb_launch.h"

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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
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

__device__ __forceinline__ void store_row4(float* base, long long p, int i0, int nx, float4 v) {
  if (i0 + 3 < nx) {
    *reinterpret_cast<float4*>(base + p) = v;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + q < nx) base[p + q] = elc(v, q);
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
__global__ void __launch_bounds__(kThreads, 1)
    k_fused(const __grid_constant__ FusedArgs a, const __grid_constant__ TMaps tm) {
  constexpr int NARR = 6 + CAC + CBC + DAC + DBC;
  constexpr int S_CA = 6, S_CB = 6 + CAC, S_DA = 6 + CAC + CBC, S_DB = 6 + CAC + CBC + DAC;
  extern __shared__ __align__(128) float smem[];

  const Geo& g = a.g;
  const CoefArgs& co = a.co;
  const int S = a.nstages;
  float* stages = smem;
  float* enew = smem + (size_t)S * NARR * kSlot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(enew + 9 * kEPlane);

  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int kz0 = blockIdx.z * a.zchunk;
  const int kz1 = min(kz0 + a.zchunk, g.nz);
  const bool top = (kz1 == g.nz);
  const int kend = top ? g.nz - 1 : kz1;  // non-top chunks stream plane kz1 for E(kz1)
  const int L = kend - kz0 + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int it) {
    const int s = it % S;
    const uint32_t bar = smem_u32(&bars[s]);
    mbar_expect_tx(bar, (uint32_t)(NARR * kBX * kBY * 4));
#pragma unroll
    for (int q = 0; q < NARR; ++q)
      tma_load_3d(smem_u32(stages + ((size_t)s * NARR + q) * kSlot), &tm.m[q], x0 - 4, y0 - 1,
                  kz0 + it, bar);
  };
  if (threadIdx.x == 0) {
    const int n0 = S < L ? S : L;
    for (int it = 0; it < n0; ++it) issue(it);
  }

  const int j = y0 + w;  // w == kTY: the +y halo row
  const int i0 = x0 + 4 * l;
  const int ih = x0 + kTX;  // +x halo column (lane 31 only)
  const int r = w + 1, c = 4 + 4 * l;
  const bool hl = (l == 31);

  // Per-thread constants: axis coefficients and masks.
  const float cdy_e = co.cdy_e[j], cdy_h = co.cdy_h[j];
  const float4 cdx_e = ldg4(co.cdx_e + i0), cdx_h = ldg4(co.cdx_h + i0);
  const float cdx_e_h = co.cdx_e[ih];
  const bool jin = j >= 1 && j < g.ny, jlt = j < g.ny;

  // H of plane k-1 at the positions this thread updates (prologue: kz0-1).
  float4 phx = make_float4(0.f, 0.f, 0.f, 0.f), phy = phx, phz = phx, pda = phx, pdb = phx;
  float hph_x = 0.f, hph_y = 0.f;  // halo column hx, hy (lane 31)
  if (kz0 > 0 && j <= g.ny) {
    const long long p = gidx(g, i0, j, kz0 - 1);
    phx = ldg4(a.in[3] + p);
    phy = ldg4(a.in[4] + p);
    if (hl && ih <= g.nx) {
      const long long ph = gidx(g, ih, j, kz0 - 1);
      hph_x = __ldg(a.in[3] + ph);
      hph_y = __ldg(a.in[4] + ph);
    }
  }

  auto h_phase = [&](int kh, const float* ep, float4 exk, float4 eyk) {
    // ep: E^{n+1} plane kh (3 comps, pitch kEW). exk/eyk: own E^{n+1} at kh+1.
    const float* pex = ep;
    const float* pey = ep + kEPlane;
    const float* pez = ep + 2 * kEPlane;
    const float4 ex_h = lds4(pex + w * kEW + 4 * l);
    const float4 ex_jp = lds4(pex + (w + 1) * kEW + 4 * l);
    const float4 ey_h = lds4(pey + w * kEW + 4 * l);
    const float4 ey_ip = shift_ip(ey_h, l, pey[w * kEW + kTX]);
    const float4 ez_h = lds4(pez + w * kEW + 4 * l);
    const float4 ez_jp = lds4(pez + (w + 1) * kEW + 4 * l);
    const float4 ez_ip = shift_ip(ez_h, l, pez[w * kEW + kTX]);
    const float cdz_h = co.cdz_h[kh];
    float4 hx, hy, hz;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float A = DAC ? elc(pda, q) : co.da_s;
      const float B = elc(pdb, q);
      // hx(i,j,k) += cdz[k]*(ey(k+1)-ey(k)) - cdy[j]*(ez(j+1)-ez(j))
      el(hx, q) = yee_upd(A, elc(phx, q), DBC ? B : cdz_h, elc(eyk, q), elc(ey_h, q),
                          DBC ? B : cdy_h, elc(ez_jp, q), elc(ez_h, q));
      // hy(i,j,k) += cdx[i]*(ez(i+1)-ez(i)) - cdz[k]*(ex(k+1)-ex(k))
      el(hy, q) = yee_upd(A, elc(phy, q), DBC ? B : elc(cdx_h, q), elc(ez_ip, q), elc(ez_h, q),
                          DBC ? B : cdz_h, elc(exk, q), elc(ex_h, q));
      // hz(i,j,k) += cdy[j]*(ex(j+1)-ex(j)) - cdx[i]*(ey(i+1)-ey(i))
      el(hz, q) = yee_upd(A, elc(phz, q), DBC ? B : cdy_h, elc(ex_jp, q), elc(ex_h, q),
                          DBC ? B : elc(cdx_h, q), elc(ey_ip, q), elc(ey_h, q));
    }
    if (jlt) {
      const long long p = gidx(g, i0, j, kh);
      store_row4(a.out[3], p, i0, g.nx, hx);
      store_row4(a.out[4], p, i0, g.nx, hy);
      store_row4(a.out[5], p, i0, g.nx, hz);
    }
  };

  float4 exn, eyn;
  for (int it = 0; it < L; ++it) {
    const int k = kz0 + it;
    const int s = it % S;
    mbar_wait(smem_u32(&bars[s]), (uint32_t)((it / S) & 1));
    const float* st = stages + (size_t)s * NARR * kSlot;
#define SM(q, rr, cc) (st + (q) * kSlot + (rr) * kBX + (cc))

    // ---------------- E phase: plane k, rows y0..y0+TY, cols x0..x0+TX ----
    const float cdz_e = co.cdz_e[k];
    const bool kin = k >= 1 && k < g.nz;
    const float4 ex = lds4(SM(0, r, c)), ey = lds4(SM(1, r, c)), ez = lds4(SM(2, r, c));
    const float4 hx = lds4(SM(3, r, c)), hx_jm = lds4(SM(3, r - 1, c));
    const float4 hy = lds4(SM(4, r, c));
    const float4 hz = lds4(SM(5, r, c)), hz_jm = lds4(SM(5, r - 1, c));
    const float4 hy_im = shift_im(hy, l, *SM(4, r, c - 1));
    const float4 hz_im = shift_im(hz, l, *SM(5, r, c - 1));
    float4 ca4 = make_float4(0.f, 0.f, 0.f, 0.f), cb4 = ca4;
    if (CAC) ca4 = lds4(SM(S_CA, r, c));
    if (CBC) cb4 = lds4(SM(S_CB, r, c));
    float4 ezn;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q;
      const float A = CAC ? elc(ca4, q) : co.ca_s;
      const float B = elc(cb4, q);
      const bool iin = i >= 1 && i < g.nx;
      el(exn, q) = (i < g.nx && jin && kin)
                       ? yee_upd(A, elc(ex, q), CBC ? B : cdy_e, elc(hz, q), elc(hz_jm, q),
                                 CBC ? B : cdz_e, elc(hy, q), elc(phy, q))
                       : 0.f;
      el(eyn, q) = (iin && jlt && kin)
                       ? yee_upd(A, elc(ey, q), CBC ? B : cdz_e, elc(hx, q), elc(phx, q),
                                 CBC ? B : elc(cdx_e, q), elc(hz, q), elc(hz_im, q))
                       : 0.f;
      el(ezn, q) = (iin && jin)
                       ? yee_upd(A, elc(ez, q), CBC ? B : elc(cdx_e, q), elc(hy, q),
                                 elc(hy_im, q), CBC ? B : cdy_e, elc(hx, q), elc(hx_jm, q))
                       : 0.f;
    }
    // soft sources (after PEC, before Faraday): comp(i,j,k) += val
    for (int q = 0; q < a.src.n; ++q) {
      if (a.src.k[q] != k || a.src.j[q] != j) continue;
      const int d = a.src.i[q] - i0;
      const float v = a.src.val[q];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (d != e) continue;
        if (a.src.comp[q] == 0) el(exn, e) = __fadd_rn(el(exn, e), v);
        if (a.src.comp[q] == 1) el(eyn, e) = __fadd_rn(el(eyn, e), v);
        if (a.src.comp[q] == 2) el(ezn, e) = __fadd_rn(el(ezn, e), v);
      }
    }
    float* eb = enew + (it % 3) * 3 * kEPlane;
    sts4(eb + w * kEW + 4 * l, exn);
    sts4(eb + kEPlane + w * kEW + 4 * l, eyn);
    sts4(eb + 2 * kEPlane + w * kEW + 4 * l, ezn);
    // +x halo column i = x0+TX (lane 31): scalar form of the same update
    float hh_x = 0.f, hh_y = 0.f;
    if (hl) {
      const int cc = 4 + kTX;
      const float A = CAC ? *SM(S_CA, r, cc) : co.ca_s;
      const float B = CBC ? *SM(S_CB, r, cc) : 0.f;
      hh_x = *SM(3, r, cc);
      hh_y = *SM(4, r, cc);
      const float hzc = *SM(5, r, cc);
      const bool iin = ih >= 1 && ih < g.nx;
      float vx = (ih < g.nx && jin && kin)
                     ? yee_upd(A, *SM(0, r, cc), CBC ? B : cdy_e, hzc, *SM(5, r - 1, cc),
                               CBC ? B : cdz_e, hh_y, hph_y)
                     : 0.f;
      float vy = (iin && jlt && kin)
                     ? yee_upd(A, *SM(1, r, cc), CBC ? B : cdz_e, hh_x, hph_x,
                               CBC ? B : cdx_e_h, hzc, hz.w)
                     : 0.f;
      float vz = (iin && jin) ? yee_upd(A, *SM(2, r, cc), CBC ? B : cdx_e_h, hh_y, hy.w,
                                        CBC ? B : cdy_e, hh_x, *SM(3, r - 1, cc))
                              : 0.f;
      for (int q = 0; q < a.src.n; ++q) {
        if (a.src.k[q] != k || a.src.j[q] != j || a.src.i[q] != ih) continue;
        if (a.src.comp[q] == 0) vx = __fadd_rn(vx, a.src.val[q]);
        if (a.src.comp[q] == 1) vy = __fadd_rn(vy, a.src.val[q]);
        if (a.src.comp[q] == 2) vz = __fadd_rn(vz, a.src.val[q]);
      }
      eb[w * kEW + kTX] = vx;
      eb[kEPlane + w * kEW + kTX] = vy;
      eb[2 * kEPlane + w * kEW + kTX] = vz;
    }
    if (w < kTY && jlt && k < kz1) {
      const long long p = gidx(g, i0, j, k);
      store_row4(a.out[0], p, i0, g.nx, exn);
      store_row4(a.out[1], p, i0, g.nx, eyn);
      store_row4(a.out[2], p, i0, g.nx, ezn);
    }
    // H and coefficients of plane k at own positions, for the next H phase
    float4 chz = hz;
    float4 cda = pda, cdb = pdb;
    if (DAC) cda = lds4(SM(S_DA, r, c));
    if (DBC) cdb = lds4(SM(S_DB, r, c));
#undef SM
    __syncthreads();  // E plane k complete; stage s free for refill
    if (threadIdx.x == 0 && it + S < L) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + S);
    }
    // ---------------- H phase: plane k-1 ------------------------------------
    if (it >= 1 && w < kTY) h_phase(k - 1, enew + ((it - 1) % 3) * 3 * kEPlane, exn, eyn);
    phx = hx;
    phy = hy;
    phz = chz;
    pda = cda;
    pdb = cdb;
    hph_x = hh_x;
    hph_y = hh_y;
  }
  // top chunk: H on plane nz-1 sees the PEC zeros of ex/ey at plane nz
  if (top && w < kTY) {
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    h_phase(g.nz - 1, enew + ((L - 1) % 3) * 3 * kEPlane, z4, z4);
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t launch_t(const FusedArgs& a, const TMaps& tm, dim3 grid, size_t smem, cudaStream_t st) {
  k_fused<CAC, CBC, DAC, DBC><<<grid, kThreads, smem, st>>>(a, tm);
  return cudaGetLastError();
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t set_limit_t() {
  return cudaFuncSetAttribute(k_fused<CAC, CBC, DAC, DBC>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

using LaunchFn = cudaError_t (*)(const FusedArgs&, const TMaps&, dim3, size_t, cudaStream_t);
using LimitFn = cudaError_t (*)();

#define YB_T(m) launch_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0>
#define YB_L(m) set_limit_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0>
const LaunchFn kLaunch[16] = {YB_T(0),  YB_T(1),  YB_T(2),  YB_T(3), YB_T(4),  YB_T(5),
                              YB_T(6),  YB_T(7),  YB_T(8),  YB_T(9), YB_T(10), YB_T(11),
                              YB_T(12), YB_T(13), YB_T(14), YB_T(15)};
const LimitFn kLimit[16] = {YB_L(0),  YB_L(1),  YB_L(2),  YB_L(3), YB_L(4),  YB_L(5),
                            YB_L(6),  YB_L(7),  YB_L(8),  YB_L(9), YB_L(10), YB_L(11),
                            YB_L(12), YB_L(13), YB_L(14), YB_L(15)};
#undef YB_T
#undef YB_L

}  // namespace

cudaError_t fused_set_smem_limits() {
  for (int m = 0; m < 16; ++m) {
    const cudaError_t e = kLimit[m]();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_fused(const FusedArgs& a, const TMaps& tm, int cell_mask, dim3 grid,
                         size_t smem, cudaStream_t st) {
  return kLaunch[cell_mask & 15](a, tm, grid, smem, st);
}

}  // namespace yb
