// yb_fused.cu — the FUSED one-sweep Yee step for sm_100a.
//
// Work item = a kTX x kTY column of cells (x,y) times a z-chunk of planes.
// Persistent CTAs (one per SM) take items from a global atomic counter.
// Warp kTY is the producer: one lane streams, per plane, a box
// x0-4..x0+TX+3, y0-1..y0+TY of every read array (ex..hz of the current
// state + the per-cell coefficient arrays) into a ring of `nstages` shared
// stages with cp.async.bulk.tensor, completion on a "full" mbarrier.
// Warps 0..kTY-1 are independent z-marching row units: warp w owns row
// j = y0+w and per plane k
//   1. computes E^{n+1}(k) on row j (update_e_dof, kernels.hpp:27-44, PEC
//      folded in as "not curl-updatable -> +0", staggering.hpp:70-86,
//      sources added after it, schedule.hpp:175-199), plus the E values of
//      the +y row (ex, ez) and +x column (ey, ez) that its H update needs -
//      recomputed redundantly, so no warp ever waits for another;
//   2. releases the stage (one arrive per warp on the "empty" mbarrier);
//   3. computes H^{n+3/2}(k-1) on row j (update_h_dof, kernels.hpp:46-63)
//      from registers only: E(k-1) with its halo, E(k), H(k-1), Da/Db(k-1).
// Warp kTY+1 updates the DoFs of the three upper faces (face_point)
// concurrently, so one launch performs the whole Standard step.
// This is planeAmpere(k); planeFaraday(k-1) of the paper's one-sweep scheme
// (PAPER.md:683-692).
// State is double-buffered (read `in`, write `out`), so CTAs never race on
// halo values; DRAM traffic is one read + one write of each field plus one
// read of each per-cell coefficient array per step.
// Arithmetic: yee_upd (explicit _rn intrinsics), bit-identical to the oracle.
#include <cuda.h>
#include <cuda_runtime.h>

#include "yb_launch.h"
#include "yb_ptx.cuh"

namespace yb {
namespace {

template <bool CAC, bool CBC, bool DAC, bool DBC, bool QS>
__global__ void __launch_bounds__(kThreads, 1)
    k_fused(const __grid_constant__ FusedArgs a, const __grid_constant__ TMaps tm) {
  constexpr int NARR = 6 + CAC + CBC + DAC + DBC;
  constexpr int S_CA = 6, S_CB = 6 + CAC, S_DA = 6 + CAC + CBC, S_DB = 6 + CAC + CBC + DAC;
  constexpr uint32_t kBoxBytes = kBX * kBY * 4;
  constexpr int kQ = 8;  // item queue depth (> max stages)
  extern __shared__ __align__(128) float smem[];

  const Geo& g = a.g;
  const CoefArgs& co = a.co;
  const int S = a.nstages;
  float* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * NARR * kSlot);
  uint64_t* empty = full + S;
  int* item_q = reinterpret_cast<int*>(empty + S);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int T = a.ntx * a.nty;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kTY);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ======================= producer warp ===================================
  // Items are numbered chunk-major and handed out in order, so the items in
  // flight form a contiguous window: concurrently running CTAs hold
  // neighbouring tiles at the same z and their halo rows meet in L2.
  // Element 0 of an item with kz0 > 0 is the prologue plane kz0-1 (hx, hy
  // only); then planes kz0..kend. The item index reaches the consumers
  // through item_q, published by the (release) arrive on the item's first
  // full barrier; -1 (no work left) is published by a plain arrive.
  if (w == kTY + 1) {  // face warp: the upper-face DoFs (face_point)
    if (a.no_faces) return;
    const long long nf = face_points(g);
    for (long long t = blockIdx.x * 32LL + l; t < nf; t += gridDim.x * 32LL)
      face_point(g, a.in, a.out, co, t);
    return;
  }
  if (w == kTY) {
    if (l != 0) return;
    int p_item = -1, p_e = 0, p_nE = 0, p_seq = 0;
    for (int q = 0;; ++q) {
      const int s = q % S;
      if (q >= S) mbar_wait(smem_u32(&empty[s]), (uint32_t)(((q / S) - 1) & 1));
      const uint32_t bar = smem_u32(&full[s]);
      if (p_item < 0) {
        const unsigned long long v = atomicAdd(a.sched, 1ull) - a.sched_base;
        const int it = v < (unsigned long long)a.nitems ? (int)v : -1;
        item_q[p_seq % kQ] = it;
        ++p_seq;
        if (it < 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
          return;
        }
        int kz0, kz1;
        chunk_planes(a, it / T, kz0, kz1);
        const bool pro = kz0 > 0 || !at_bottom(g);
        const int kend = (kz1 == g.nz && at_top(g)) ? g.nz - 1 : kz1;
        if (QS) {  // quiescent item: input box all +0, no source -> skip
          const int tl = it % T, tx = tl % a.ntx, ty = tl / a.ntx;
          const int x0 = tx * kTX, y0 = ty * kTY;
          if (!src_in_box(a.src, x0 - 4, x0 + kTX + 3, y0 - 1, y0 + kTY, kz0 - 1, kend) &&
              !qmap_dirty(a.qm, tx, ty, kz0 - 1, kend)) {
            item_q[(p_seq - 1) % kQ] = it | kSkipItem;
            atomicAdd(a.skipped, 1ull);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
            continue;  // the item occupies this one (empty) stage
          }
        }
        p_item = it;
        p_e = 0;
        p_nE = (pro ? 1 : 0) + kend - kz0 + 1;
      }
      const int chunk = p_item / T, tile = p_item - chunk * T;
      const int x0 = (tile % a.ntx) * kTX, y0 = (tile / a.ntx) * kTY;
      int kz0, kz1_unused;
      chunk_planes(a, chunk, kz0, kz1_unused);
      const int pro = (kz0 > 0 || !at_bottom(g)) ? 1 : 0;
      float* dst = stages + (size_t)s * NARR * kSlot;
      // tensor z coordinate = local plane + kGhost (ghost plane -kGhost is z = 0)
      if (pro && p_e == 0) {
        mbar_expect_tx(bar, 2 * kBoxBytes);
        tma_load_3d(smem_u32(dst + 3 * kSlot), &tm.m[3], x0 - 4, y0 - 1, kz0 - 1 + kGhost, bar);
        tma_load_3d(smem_u32(dst + 4 * kSlot), &tm.m[4], x0 - 4, y0 - 1, kz0 - 1 + kGhost, bar);
      } else {
        const int k = kz0 + p_e - pro;
        mbar_expect_tx(bar, NARR * kBoxBytes);
#pragma unroll
        for (int qq = 0; qq < NARR; ++qq)
          tma_load_3d(smem_u32(dst + qq * kSlot), &tm.m[qq], x0 - 4, y0 - 1, k + kGhost, bar);
      }
      if (++p_e == p_nE) p_item = -1;
    }
  }

  // ======================= consumer warps ==================================
  uint64_t st_pol;
  if (a.store_policy == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(st_pol));
  else if (a.store_policy == 2)
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(st_pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(st_pol));
  const int r = w + 1, rn = w + 2, c = 4 + 4 * l;  // smem row of j, j+1; col of i0
  const bool hl = (l == 31);
  constexpr int cc = 4 + kTX;  // smem col of the +x halo column
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  int cs = 0, c_seq = 0;
  bool peeked = false;
  auto wait_elem = [&]() -> int {
    const int s = cs % S;
    if (!peeked) mbar_wait(smem_u32(&full[s]), (uint32_t)((cs / S) & 1));
    peeked = false;
    ++cs;
    return s;
  };
  auto release = [&](int s) {
    __syncwarp();
    if (l == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                             : "memory");
  };

  for (;;) {
    mbar_wait(smem_u32(&full[cs % S]), (uint32_t)((cs / S) & 1));
    peeked = true;
    const int item = item_q[c_seq % kQ];
    ++c_seq;
    if (item < 0) break;
    if (QS && (item & kSkipItem)) {  // quiescent: consume the empty stage, nothing to write
      release(wait_elem());
      continue;
    }
    const int chunk = item / T, tile = item - chunk * T;
    const int x0 = (tile % a.ntx) * kTX, y0 = (tile / a.ntx) * kTY;
    int kz0, kz1;
    chunk_planes(a, chunk, kz0, kz1);
    const bool top = (kz1 == g.nz) && at_top(g);  // global top: E(nz) is PEC
    const int kend = top ? g.nz - 1 : kz1;      // else stream plane kz1 (maybe the ghost)

    const int j = y0 + w, jn = j + 1;
    const int i0 = x0 + 4 * l;
    const int ih = x0 + kTX;  // +x halo column (lane 31)
    const float cdy_e = co.cdy_e[j], cdy_en = co.cdy_e[jn], cdy_h = co.cdy_h[j];
    const float4 cdx_e = ldg4(co.cdx_e + i0), cdx_h = ldg4(co.cdx_h + i0);
    const float cdx_e_h = co.cdx_e[ih];
    const bool jin = j >= 1 && j < g.ny, jlt = j < g.ny;
    const bool jnin = jn < g.ny;  // jn >= 1 always
    const bool ih_in = ih >= 1 && ih < g.nx;
    const bool xint = i0 >= 1 && i0 + 4 <= g.nx;  // this lane touches neither i=0 nor i>=nx

    // carried state: H(k-1) (own row, hy of row j+1, hx of the halo column),
    // Da/Db(k-1), E(k-1) own row / +y row (ex, ez) / +x column (ey, ez)
    float4 phx = z4, phy = z4, phz = z4, phy_n = z4, pda = z4, pdb = z4;
    float phx_c = 0.f;
    float4 pex = z4, pey = z4, pez = z4, pex_n = z4, pez_n = z4;
    float pey_c = 0.f, pez_c = 0.f;

    auto h_row = [&](int kh, float4 exk, float4 eyk) {
      const float4 ey_ip = shift_ip(pey, l, pey_c);
      const float4 ez_ip = shift_ip(pez, l, pez_c);
      const float cdz_h = co.cdz_h[kh];
      float4 hx, hy, hz;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float A = DAC ? elc(pda, q) : co.da_s;
        const float B = elc(pdb, q);
        // hx(i,j,k) += cdz[k]*(ey(k+1)-ey(k)) - cdy[j]*(ez(j+1)-ez(j))
        el(hx, q) = yee_upd_t<DAC>(A, elc(phx, q), DBC ? B : cdz_h, elc(eyk, q), elc(pey, q),
                            DBC ? B : cdy_h, elc(pez_n, q), elc(pez, q));
        // hy(i,j,k) += cdx[i]*(ez(i+1)-ez(i)) - cdz[k]*(ex(k+1)-ex(k))
        el(hy, q) = yee_upd_t<DAC>(A, elc(phy, q), DBC ? B : elc(cdx_h, q), elc(ez_ip, q), elc(pez, q),
                            DBC ? B : cdz_h, elc(exk, q), elc(pex, q));
        // hz(i,j,k) += cdy[j]*(ex(j+1)-ex(j)) - cdx[i]*(ey(i+1)-ey(i))
        el(hz, q) = yee_upd_t<DAC>(A, elc(phz, q), DBC ? B : cdy_h, elc(pex_n, q), elc(pex, q),
                            DBC ? B : elc(cdx_h, q), elc(ey_ip, q), elc(pey, q));
      }
      if (jlt) {
        const long long p = gidx(g, i0, j, kh);
        store_rows3(a.out + 3, p, i0, g.nx, hx, hy, hz, st_pol);
      }
      if (QS && __any_sync(~0u, jlt && (nonzero4(hx) | nonzero4(hy) | nonzero4(hz))) && l == 0)
        qmap_mark(a.qm, tile, kh);
    };

    if (kz0 > 0 || !at_bottom(g)) {  // prologue element: H^{n+1/2} on plane kz0-1
      const int s = wait_elem();
      const float* st = stages + (size_t)s * NARR * kSlot;
      phx = lds4(st + 3 * kSlot + r * kBX + c);
      phy = lds4(st + 4 * kSlot + r * kBX + c);
      phy_n = lds4(st + 4 * kSlot + rn * kBX + c);
      if (hl) phx_c = st[3 * kSlot + r * kBX + cc];
      release(s);
    }

    for (int k = kz0; k <= kend; ++k) {
      const int s = wait_elem();
      const float* st = stages + (size_t)s * NARR * kSlot;
#define SM(q, rr, col) (st + (q) * kSlot + (rr) * kBX + (col))
      const float cdz_e = co.cdz_e[k];
      const int kg = k + g.zoff;  // global plane (PEC at global z = 0, nzg)
      const bool kin = kg >= 1 && kg < g.nzg;
      // own row j
      const float4 ex = lds4(SM(0, r, c)), ey = lds4(SM(1, r, c)), ez = lds4(SM(2, r, c));
      const float4 hx = lds4(SM(3, r, c)), hy = lds4(SM(4, r, c)), hz = lds4(SM(5, r, c));
      const float4 hx_jm = lds4(SM(3, r - 1, c)), hz_jm = lds4(SM(5, r - 1, c));
      const float4 hy_im = shift_im(hy, l, *SM(4, r, c - 1));
      const float4 hz_im = shift_im(hz, l, *SM(5, r, c - 1));
      // +y row j+1 (ex, ez only)
      const float4 ex_n = lds4(SM(0, rn, c)), ez_n = lds4(SM(2, rn, c));
      const float4 hx_n = lds4(SM(3, rn, c)), hy_n = lds4(SM(4, rn, c)), hz_n = lds4(SM(5, rn, c));
      const float4 hy_n_im = shift_im(hy_n, l, *SM(4, rn, c - 1));
      float4 ca4 = z4, cb4 = z4, ca4n = z4, cb4n = z4, da4 = pda, db4 = pdb;
      if (CAC) {
        ca4 = lds4(SM(S_CA, r, c));
        ca4n = lds4(SM(S_CA, rn, c));
      }
      if (CBC) {
        cb4 = lds4(SM(S_CB, r, c));
        cb4n = lds4(SM(S_CB, rn, c));
      }
      if (DAC) da4 = lds4(SM(S_DA, r, c));
      if (DBC) db4 = lds4(SM(S_DB, r, c));
      float4 exw, eyw, ezw, exn, ezn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // unmasked updates; PEC / non-DoF zeroed below
        const float A = CAC ? elc(ca4, q) : co.ca_s;
        const float B = elc(cb4, q);
        const float An = CAC ? elc(ca4n, q) : co.ca_s;
        const float Bn = elc(cb4n, q);
        el(exw, q) = yee_upd_t<CAC>(A, elc(ex, q), CBC ? B : cdy_e, elc(hz, q), elc(hz_jm, q), CBC ? B : cdz_e,
                             elc(hy, q), elc(phy, q));
        el(eyw, q) = yee_upd_t<CAC>(A, elc(ey, q), CBC ? B : cdz_e, elc(hx, q), elc(phx, q),
                             CBC ? B : elc(cdx_e, q), elc(hz, q), elc(hz_im, q));
        el(ezw, q) = yee_upd_t<CAC>(A, elc(ez, q), CBC ? B : elc(cdx_e, q), elc(hy, q), elc(hy_im, q),
                             CBC ? B : cdy_e, elc(hx, q), elc(hx_jm, q));
        el(exn, q) = yee_upd_t<CAC>(An, elc(ex_n, q), CBC ? Bn : cdy_en, elc(hz_n, q), elc(hz, q),
                             CBC ? Bn : cdz_e, elc(hy_n, q), elc(phy_n, q));
        el(ezn, q) = yee_upd_t<CAC>(An, elc(ez_n, q), CBC ? Bn : elc(cdx_e, q), elc(hy_n, q), elc(hy_n_im, q),
                             CBC ? Bn : cdy_en, elc(hx_n, q), elc(hx, q));
      }
      if (!(xint && jin && jnin && kin)) {  // only lanes on a boundary column/row/plane
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = i0 + q;
          const bool iin = i >= 1 && i < g.nx, ilt = i < g.nx;
          if (!(ilt && jin && kin)) el(exw, q) = 0.f;
          if (!(iin && jlt && kin)) el(eyw, q) = 0.f;
          if (!(iin && jin)) el(ezw, q) = 0.f;
          if (!(ilt && jnin && kin)) el(exn, q) = 0.f;
          if (!(iin && jnin)) el(ezn, q) = 0.f;
        }
      }
      // +x halo column i = x0+TX, row j: ey, ez (lane 31)
      float eyc = 0.f, ezc = 0.f, hx_c = 0.f;
      if (hl) {
        const float A = CAC ? *SM(S_CA, r, cc) : co.ca_s;
        const float B = CBC ? *SM(S_CB, r, cc) : 0.f;
        hx_c = *SM(3, r, cc);
        const float hy_c = *SM(4, r, cc), hz_c = *SM(5, r, cc);
        eyc = (ih_in && jlt && kin) ? yee_upd_t<CAC>(A, *SM(1, r, cc), CBC ? B : cdz_e, hx_c, phx_c,
                                              CBC ? B : cdx_e_h, hz_c, hz.w)
                                    : 0.f;
        ezc = (ih_in && jin) ? yee_upd_t<CAC>(A, *SM(2, r, cc), CBC ? B : cdx_e_h, hy_c, hy.w,
                                       CBC ? B : cdy_e, hx_c, *SM(3, r - 1, cc))
                             : 0.f;
      }
#undef SM
      release(s);  // everything this warp needs from the stage is in registers
      // soft sources (after PEC, before Faraday): comp(i,j,k) += val, for
      // every copy of the DoF this warp computed
      for (int q = 0; q < a.src.n; ++q) {
        if (a.src.k[q] != k) continue;
        const int sc = a.src.comp[q], si = a.src.i[q], sj = a.src.j[q];
        const float v = a.src.val[q];
        const int d = si - i0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (d != e) continue;
          if (sj == j) {
            if (sc == 0) el(exw, e) = __fadd_rn(el(exw, e), v);
            if (sc == 1) el(eyw, e) = __fadd_rn(el(eyw, e), v);
            if (sc == 2) el(ezw, e) = __fadd_rn(el(ezw, e), v);
          }
          if (sj == jn) {
            if (sc == 0) el(exn, e) = __fadd_rn(el(exn, e), v);
            if (sc == 2) el(ezn, e) = __fadd_rn(el(ezn, e), v);
          }
        }
        if (hl && si == ih && sj == j) {
          if (sc == 1) eyc = __fadd_rn(eyc, v);
          if (sc == 2) ezc = __fadd_rn(ezc, v);
        }
      }
      if (jlt && k < kz1) {
        const long long p = gidx(g, i0, j, k);
        store_rows3(a.out, p, i0, g.nx, exw, eyw, ezw, st_pol);
      }
      if (QS && k < kz1 &&
          __any_sync(~0u, jlt && (nonzero4(exw) | nonzero4(eyw) | nonzero4(ezw))) && l == 0)
        qmap_mark(a.qm, tile, k);
      if (k > kz0) h_row(k - 1, exw, eyw);
      pex = exw;
      pey = eyw;
      pez = ezw;
      pex_n = exn;
      pez_n = ezn;
      pey_c = eyc;
      pez_c = ezc;
      phx = hx;
      phy = hy;
      phz = hz;
      phy_n = hy_n;
      phx_c = hx_c;
      pda = da4;
      pdb = db4;
    }
    // top chunk: H on plane nz-1 sees the PEC zeros of ex/ey at plane nz
    if (top) h_row(g.nz - 1, z4, z4);
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC, bool QS>
cudaError_t launch_t(const FusedArgs& a, const TMaps& tm, dim3 grid, size_t smem, cudaStream_t st) {
  k_fused<CAC, CBC, DAC, DBC, QS><<<grid, kThreads, smem, st>>>(a, tm);
  return cudaGetLastError();
}

template <bool CAC, bool CBC, bool DAC, bool DBC, bool QS>
cudaError_t set_limit_t() {
  return cudaFuncSetAttribute(k_fused<CAC, CBC, DAC, DBC, QS>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

using LaunchFn = cudaError_t (*)(const FusedArgs&, const TMaps&, dim3, size_t, cudaStream_t);
using LimitFn = cudaError_t (*)();

#define YB_T(m) launch_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0, (m & 16) != 0>
#define YB_L(m) set_limit_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0, (m & 16) != 0>
const LaunchFn kLaunch[32] = {YB_T(0),  YB_T(1),  YB_T(2),  YB_T(3),  YB_T(4),  YB_T(5),  YB_T(6),  YB_T(7),
                              YB_T(8),  YB_T(9),  YB_T(10), YB_T(11), YB_T(12), YB_T(13), YB_T(14), YB_T(15),
                              YB_T(16), YB_T(17), YB_T(18), YB_T(19), YB_T(20), YB_T(21), YB_T(22), YB_T(23),
                              YB_T(24), YB_T(25), YB_T(26), YB_T(27), YB_T(28), YB_T(29), YB_T(30), YB_T(31)};
const LimitFn kLimit[32] = {YB_L(0),  YB_L(1),  YB_L(2),  YB_L(3),  YB_L(4),  YB_L(5),  YB_L(6),  YB_L(7),
                            YB_L(8),  YB_L(9),  YB_L(10), YB_L(11), YB_L(12), YB_L(13), YB_L(14), YB_L(15),
                            YB_L(16), YB_L(17), YB_L(18), YB_L(19), YB_L(20), YB_L(21), YB_L(22), YB_L(23),
                            YB_L(24), YB_L(25), YB_L(26), YB_L(27), YB_L(28), YB_L(29), YB_L(30), YB_L(31)};
#undef YB_T
#undef YB_L

}  // namespace

cudaError_t fused_set_smem_limits() {
  for (int m = 0; m < 32; ++m) {
    const cudaError_t e = kLimit[m]();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_fused(const FusedArgs& a, const TMaps& tm, int cell_mask, dim3 grid,
                         size_t smem, cudaStream_t st) {
  return kLaunch[(cell_mask & 15) | (a.qm.bits ? 16 : 0)](a, tm, grid, smem, st);
}

}  // namespace yb
