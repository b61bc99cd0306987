// yb_tb4.cu — temporal blocking of depth 4: FOUR full Standard steps per
// sweep (eight fused half-steps E1,H1,..,E4,H4), the depth-8 point of the
// BASELINE config-5 temporal-depth sweep. It reads the state and the
// coefficients once and writes the state once per four steps (16 / 12 B per
// cell-update for 4 / 1 coefficient arrays), at the price of recomputing a
// shrinking halo at every level.
//
// Work item = 4 output rows x 56 output columns x a z-chunk. Every warp
// computes every level over a fixed 11-row x 64-column window (rows
// y0-3..y0+7, columns x0-4..x0+59, float2 per lane); the region where a level
// is valid shrinks by one row / column per half-step (E loses the lower row and
// left column it cannot see, H the upper row and right column), and after
// eight half-steps rows y0..y0+3, columns x0..x0+55 are exact. Values outside
// the valid region are computed but never stored. Per plane p the levels run
// as a wavefront: E_l at plane p-l+1, H_l at plane p-l (kernels.hpp:27-63,
// PEC folded in as masks, sources after their E level, schedule.hpp:175-199);
// every level is double-buffered in shared memory by plane parity; one CTA
// barrier before each of E2, E3, E4. A TMA producer warp streams the 12-row
// field boxes and 11-row coefficient boxes of planes pstart-1..pin_end
// (mbarrier ring); a face warp applies the four steps to the upper-face DoFs.
// Single-domain only (a z-slab would need four ghost planes). Arithmetic:
// yee_upd_t, bit-identical to four single steps.
#include <cuda.h>
#include <cuda_runtime.h>

#include "yb_launch.h"
#include "yb_ptx.cuh"

namespace yb {
namespace {

constexpr int K4 = 4;                        // steps per sweep
constexpr int R4 = kTB4Rows;                 // output rows per item
constexpr int RW4 = kTB4RowWarps;            // row warps: window rows y0-3 .. y0+7
constexpr int WC = kTB4Win;                  // window columns x0-4 .. x0+59
constexpr int PROD4 = RW4, FACE4 = RW4 + 1;  // warp roles
constexpr int LV = RW4 * WC;                 // floats of one level-plane component
constexpr int kSlots = 2 * K4 - 1;           // buffered levels: E1 H1 E2 H2 E3 H3 E4

__device__ __forceinline__ void sync_rows() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * RW4) : "memory");
}

__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

struct V3 {
  float2 x, y, z;
};

// Stage layout: fields (12 rows from y0-4), then the per-cell coefficient
// arrays present (11 rows from y0-3).
template <bool CAC, bool CBC, bool DAC, bool DBC>
struct Stage4 {
  static constexpr int F = kTB4BY * WC;        // floats per field slot
  static constexpr int C = (kTB4BY - 1) * WC;  // floats per coefficient slot
  static constexpr int floats = 6 * F + (CAC + CBC + DAC + DBC) * C;
  static constexpr int off_ca = 6 * F;
  static constexpr int off_cb = off_ca + CAC * C;
  static constexpr int off_da = off_cb + CBC * C;
  static constexpr int off_db = off_da + DAC * C;
};

struct Item4 {
  int x0, y0, kz0, kz1, pstart, pin_end, pend;
  bool pro;
};

__device__ __forceinline__ Item4 make_item4(const FusedArgs& a, int item) {
  const int T = a.ntx * a.nty;
  const int chunk = item / T, tile = item - chunk * T;
  Item4 it;
  it.x0 = (tile % a.ntx) * kTB4Cols;
  it.y0 = (tile / a.ntx) * R4;
  chunk_planes(a, chunk, it.kz0, it.kz1);
  it.pstart = max(it.kz0 - (K4 - 1), 0);
  it.pro = it.pstart > 0;
  it.pin_end = min(it.kz1 + K4 - 1, a.g.nz - 1);
  it.pend = it.kz1 + K4 - 1;
  return it;
}

// The four steps' source increments (step n + s at bit s).
struct Src4 {
  int n;
  int comp[kMaxSources], i[kMaxSources], j[kMaxSources], k[kMaxSources];
  float val[kMaxSources][K4];
  int act[kMaxSources];
};

// E update of a lane's two DoFs at (i0, i0+1), row j, global plane kg, with
// PEC / non-DoF positions forced to +0 (staggering.hpp:70-86).
template <bool CAC, bool CBC>
__device__ __forceinline__ V3 e_upd2(const CoefArgs& co, const Geo& g, int i0, int j, int kg, float cdy, float cdz,
                                     float2 cdx, float2 ca, float2 cb, const V3& e, const V3& h, float2 hx_jm,
                                     float2 hz_jm, float2 hy_im, float2 hz_im, float2 hx_km, float2 hy_km) {
  V3 o;
  const float A0 = CAC ? ca.x : co.ca_s, A1 = CAC ? ca.y : co.ca_s;
  o.x.x = yee_upd_t<CAC>(A0, e.x.x, CBC ? cb.x : cdy, h.z.x, hz_jm.x, CBC ? cb.x : cdz, h.y.x, hy_km.x);
  o.x.y = yee_upd_t<CAC>(A1, e.x.y, CBC ? cb.y : cdy, h.z.y, hz_jm.y, CBC ? cb.y : cdz, h.y.y, hy_km.y);
  o.y.x = yee_upd_t<CAC>(A0, e.y.x, CBC ? cb.x : cdz, h.x.x, hx_km.x, CBC ? cb.x : cdx.x, h.z.x, hz_im.x);
  o.y.y = yee_upd_t<CAC>(A1, e.y.y, CBC ? cb.y : cdz, h.x.y, hx_km.y, CBC ? cb.y : cdx.y, h.z.y, hz_im.y);
  o.z.x = yee_upd_t<CAC>(A0, e.z.x, CBC ? cb.x : cdx.x, h.y.x, hy_im.x, CBC ? cb.x : cdy, h.x.x, hx_jm.x);
  o.z.y = yee_upd_t<CAC>(A1, e.z.y, CBC ? cb.y : cdx.y, h.y.y, hy_im.y, CBC ? cb.y : cdy, h.x.y, hx_jm.y);
  const bool kin = kg >= 1 && kg < g.nzg, kz = kg >= 0 && kg < g.nzg;
  const bool jin = j >= 1 && j < g.ny, jlt = j >= 0 && j < g.ny;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = i0 + q;
    const bool iin = i >= 1 && i < g.nx, ilt = i >= 0 && i < g.nx;
    float& ox = q ? o.x.y : o.x.x;
    float& oy = q ? o.y.y : o.y.x;
    float& oz = q ? o.z.y : o.z.x;
    if (!(ilt && jin && kin)) ox = 0.f;
    if (!(iin && jlt && kin)) oy = 0.f;
    if (!(iin && jin && kz)) oz = 0.f;
  }
  return o;
}

// H update of a lane's two DoFs (update_h_dof, kernels.hpp:46-63).
template <bool DAC, bool DBC>
__device__ __forceinline__ V3 h_upd2(const CoefArgs& co, float cdy, float cdz, float2 cdx, float2 da, float2 db,
                                     const V3& h, const V3& e, float2 ex_jp, float2 ez_jp, float2 ey_ip,
                                     float2 ez_ip, float2 ex_kp, float2 ey_kp) {
  V3 o;
  const float A0 = DAC ? da.x : co.da_s, A1 = DAC ? da.y : co.da_s;
  o.x.x = yee_upd_t<DAC>(A0, h.x.x, DBC ? db.x : cdz, ey_kp.x, e.y.x, DBC ? db.x : cdy, ez_jp.x, e.z.x);
  o.x.y = yee_upd_t<DAC>(A1, h.x.y, DBC ? db.y : cdz, ey_kp.y, e.y.y, DBC ? db.y : cdy, ez_jp.y, e.z.y);
  o.y.x = yee_upd_t<DAC>(A0, h.y.x, DBC ? db.x : cdx.x, ez_ip.x, e.z.x, DBC ? db.x : cdz, ex_kp.x, e.x.x);
  o.y.y = yee_upd_t<DAC>(A1, h.y.y, DBC ? db.y : cdx.y, ez_ip.y, e.z.y, DBC ? db.y : cdz, ex_kp.y, e.x.y);
  o.z.x = yee_upd_t<DAC>(A0, h.z.x, DBC ? db.x : cdy, ex_jp.x, e.x.x, DBC ? db.x : cdx.x, ey_ip.x, e.y.x);
  o.z.y = yee_upd_t<DAC>(A1, h.z.y, DBC ? db.y : cdy, ex_jp.y, e.x.y, DBC ? db.y : cdx.y, ey_ip.y, e.y.y);
  return o;
}

__device__ __forceinline__ V3 ldv3(const float* p) { return {ld2(p), ld2(p + LV), ld2(p + 2 * LV)}; }
__device__ __forceinline__ void stv3(float* p, const V3& v) {
  st2(p, v.x);
  st2(p + LV, v.y);
  st2(p + 2 * LV, v.z);
}

__device__ __forceinline__ void store2(float* base, long long p, int i0, int x0, int nx, float2 v) {
  const bool a0 = i0 >= x0 && i0 < x0 + kTB4Cols && i0 < nx;
  const bool a1 = i0 + 1 >= x0 && i0 + 1 < x0 + kTB4Cols && i0 + 1 < nx;
  if (a0 && a1)
    *reinterpret_cast<float2*>(base + p) = v;
  else {
    if (a0) base[p] = v.x;
    if (a1) base[p + 1] = v.y;
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
__global__ void __maxnreg__(128) k_tb4(const __grid_constant__ FusedArgs a, const __grid_constant__ Src4 src,
                                       const __grid_constant__ TMaps tm) {
  using L = Stage4<CAC, CBC, DAC, DBC>;
  constexpr uint32_t kBytesF = L::F * 4, kBytesC = L::C * 4;
  constexpr uint32_t kStageBytes = L::floats * 4;
  constexpr int kQ = 8;
  extern __shared__ __align__(128) float smem[];
  const Geo& g = a.g;
  const CoefArgs& co = a.co;
  const int S = a.nstages;
  // [pad 32 floats][stages][pad 32][level buffers][pad 32][barriers][item queue]
  float* stages = smem + 32;
  float* lvl = stages + (size_t)S * L::floats + 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(lvl + (size_t)kSlots * 2 * 3 * LV + 32);
  uint64_t* empty = full + S;
  int* item_q = reinterpret_cast<int*>(empty + S);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), RW4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (w == FACE4) {  // upper-face DoFs: four steps of h <- Da*h + 0
    const long long nf = face_points(g);
    for (long long t = blockIdx.x * 32LL + l; t < nf; t += gridDim.x * 32LL) {
      face_point(g, a.in, a.out, co, t);
      for (int s = 1; s < K4; ++s) face_point(g, a.out, a.out, co, t);
    }
    return;
  }

  if (w == PROD4) {  // TMA producer (one lane)
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
          mbar_arrive(bar);
          return;
        }
        const Item4 pi = make_item4(a, it);
        p_item = it;
        p_e = 0;
        p_nE = (pi.pro ? 1 : 0) + pi.pin_end - pi.pstart + 1;
      }
      const Item4 pi = make_item4(a, p_item);
      const int pro = pi.pro ? 1 : 0;
      float* dst = stages + (size_t)s * L::floats;
      if (pro && p_e == 0) {  // hx, hy of plane pstart-1
        mbar_expect_tx(bar, 2 * kBytesF);
        tma_load_3d(smem_u32(dst + 3 * L::F), &tm.m[3], pi.x0 - 4, pi.y0 - 4, pi.pstart - 1 + kGhost, bar);
        tma_load_3d(smem_u32(dst + 4 * L::F), &tm.m[4], pi.x0 - 4, pi.y0 - 4, pi.pstart - 1 + kGhost, bar);
      } else {
        const int z = pi.pstart + p_e - pro + kGhost;
        mbar_expect_tx(bar, kStageBytes);
#pragma unroll
        for (int c = 0; c < 6; ++c) tma_load_3d(smem_u32(dst + c * L::F), &tm.m[c], pi.x0 - 4, pi.y0 - 4, z, bar);
        int m = 6;
        if (CAC) tma_load_3d(smem_u32(dst + L::off_ca), &tm.m[m++], pi.x0 - 4, pi.y0 - 3, z, bar);
        if (CBC) tma_load_3d(smem_u32(dst + L::off_cb), &tm.m[m++], pi.x0 - 4, pi.y0 - 3, z, bar);
        if (DAC) tma_load_3d(smem_u32(dst + L::off_da), &tm.m[m++], pi.x0 - 4, pi.y0 - 3, z, bar);
        if (DBC) tma_load_3d(smem_u32(dst + L::off_db), &tm.m[m++], pi.x0 - 4, pi.y0 - 3, z, bar);
        (void)kBytesC;
      }
      if (++p_e == p_nE) p_item = -1;
    }
  }

  // ------------------------------------------------------------ row warps
  const int r = w;                  // window row: j = y0 - 3 + r
  const int c = 2 * l;              // window column of the lane's first DoF
  int cs = 0, c_seq = 0;
  uint32_t ph = 0;
  bool peeked = false;
  auto wait_stage = [&]() -> int {
    if (!peeked) mbar_wait(smem_u32(&full[cs]), ph);
    peeked = false;
    const int s = cs;
    if (++cs == S) {
      cs = 0;
      ph ^= 1u;
    }
    return s;
  };
  auto release = [&](int s) {
    __syncwarp();
    if (l == 0) mbar_arrive(smem_u32(&empty[s]));
  };
  // level buffer of slot sl (E1=0, H1=1, .., E4=6), plane parity par, component 0, row rr, column c
  auto LB = [&](int sl, int par, int rr) { return lvl + (size_t)((sl * 2 + par) * 3) * LV + rr * WC + c; };
  const float2 z2 = f2(0.f, 0.f);

  for (;;) {
    mbar_wait(smem_u32(&full[cs]), ph);
    peeked = true;
    const int item = item_q[c_seq % kQ];
    ++c_seq;
    if (item < 0) break;
    const Item4 it = make_item4(a, item);
    const int j = it.y0 - 3 + r;
    const int i0 = it.x0 - 4 + c;
    const int jc = min(max(j, 0), g.ny - 1), ic = min(max(i0, 0), g.nx - 1), ic1 = min(max(i0 + 1, 0), g.nx - 1);
    const float cdy_e = co.cdy_e[jc], cdy_h = co.cdy_h[jc];
    const float2 cdx_e = f2(co.cdx_e[ic], co.cdx_e[ic1]), cdx_h = f2(co.cdx_h[ic], co.cdx_h[ic1]);
    // coefficient history: E level l at plane p-l+1 uses caH[l-1]; H level l at plane p-l uses daH[l]
    float2 caH[K4], cbH[K4], daH[K4 + 1], dbH[K4 + 1];
#pragma unroll
    for (int q = 0; q < K4; ++q) caH[q] = cbH[q] = z2;
#pragma unroll
    for (int q = 0; q <= K4; ++q) daH[q] = dbH[q] = z2;
    V3 h0p = {z2, z2, z2};  // H0 of plane p-1, own row
    bool src_item = false;
    for (int q = 0; q < src.n; ++q)
      src_item |= src.act[q] != 0 && src.i[q] >= it.x0 - 4 && src.i[q] < it.x0 - 4 + WC && src.j[q] >= it.y0 - 3 &&
                  src.j[q] < it.y0 - 3 + RW4 && src.k[q] >= it.pstart && src.k[q] <= it.pend;
    auto add_src = [&](V3& e, int step, int kl) {  // soft sources of step n+step on plane kl, row j
      for (int q = 0; q < src.n; ++q) {
        if (!((src.act[q] >> step) & 1) || src.j[q] != j || src.k[q] != kl) continue;
        const int d = src.i[q] - i0;
        if (d < 0 || d > 1) continue;
        const float v = src.val[q][step];
        float2& t = src.comp[q] == 0 ? e.x : (src.comp[q] == 1 ? e.y : e.z);
        if (d == 0)
          t.x = __fadd_rn(t.x, v);
        else
          t.y = __fadd_rn(t.y, v);
      }
    };

    if (it.pro) {  // prologue: hx, hy of plane pstart-1
      const int s = wait_stage();
      const float* F = stages + (size_t)s * L::floats + (r + 1) * WC + c;
      h0p.x = ld2(F + 3 * L::F);
      h0p.y = ld2(F + 4 * L::F);
      release(s);
    }

    for (int p = it.pstart; p <= it.pend; ++p) {
      const int P = p & 1;
      // ---------------------------------------------------- E1(p)
      const bool l1 = p <= it.pin_end;
      V3 ekp = {z2, z2, z2};  // E_l at plane q+1 (own row) for H_l(q)
      V3 h0n = {z2, z2, z2};
      float2 can = z2, cbn = z2, dan = z2, dbn = z2;
      if (l1) {
        const int s = wait_stage();
        const float* F = stages + (size_t)s * L::floats;
        const float* Fr = F + (r + 1) * WC + c;  // field row of j
        const float* Fc = F + r * WC + c;        // coefficient row of j
        h0n = {ld2(Fr + 3 * L::F), ld2(Fr + 4 * L::F), ld2(Fr + 5 * L::F)};
        if (CAC) can = ld2(Fc + L::off_ca);
        if (CBC) cbn = ld2(Fc + L::off_cb);
        if (DAC) dan = ld2(Fc + L::off_da);
        if (DBC) dbn = ld2(Fc + L::off_db);
        const V3 e0 = {ld2(Fr), ld2(Fr + L::F), ld2(Fr + 2 * L::F)};
        const float2 hy_im = f2(Fr[4 * L::F - 1], h0n.y.x), hz_im = f2(Fr[5 * L::F - 1], h0n.z.x);
        ekp = e_upd2<CAC, CBC>(co, g, i0, j, p + g.zoff, cdy_e, co.cdz_e[p], cdx_e, can, cbn, e0, h0n,
                               ld2(Fr + 3 * L::F - WC), ld2(Fr + 5 * L::F - WC), hy_im, hz_im, h0p.x, h0p.y);
        if (src_item) add_src(ekp, 0, p);
        stv3(LB(0, P, r), ekp);
        release(s);
      }
      // shift the coefficient history: plane p's values enter
#pragma unroll
      for (int q = K4 - 1; q > 0; --q) caH[q] = caH[q - 1], cbH[q] = cbH[q - 1];
      caH[0] = can, cbH[0] = cbn;
#pragma unroll
      for (int q = K4; q > 0; --q) daH[q] = daH[q - 1], dbH[q] = dbH[q - 1];
      daH[0] = dan, dbH[0] = dbn;

      // levels H1, E2, H2, E3, H3, E4, H4
#pragma unroll
      for (int lv = 1; lv <= K4; ++lv) {
        // ----------------------------------------------- H_lv(q), q = p - lv
        const int qh = p - lv;
        V3 hcur = {z2, z2, z2};
        const bool do_h = qh >= it.pstart;
        if (do_h) {
          const int Q = qh & 1;
          const float* e = LB(2 * (lv - 1), Q, r);  // E_lv(qh), row j
          const V3 ec = ldv3(e);
          const float2 ex_jp = ld2(e + WC), ez_jp = ld2(e + 2 * LV + WC);
          const float2 ey_ip = f2(ec.y.y, e[LV + 2]), ez_ip = f2(ec.z.y, e[2 * LV + 2]);
          const V3 hprev = lv == 1 ? h0p : ldv3(LB(2 * lv - 3, Q, r));  // H_{lv-1}(qh)
          hcur = h_upd2<DAC, DBC>(co, cdy_h, co.cdz_h[qh], cdx_h, daH[lv], dbH[lv], hprev, ec, ex_jp, ez_jp, ey_ip,
                                  ez_ip, ekp.x, ekp.y);
          if (lv < K4) {
            stv3(LB(2 * lv - 1, Q, r), hcur);
          } else if (qh >= it.kz0 && qh < it.kz1 && r >= K4 - 1 && r < K4 - 1 + R4 && j < g.ny) {
            const long long gp = gidx(g, i0, j, qh);
            store2(a.out[3], gp, i0, it.x0, g.nx, hcur.x);
            store2(a.out[4], gp, i0, it.x0, g.nx, hcur.y);
            store2(a.out[5], gp, i0, it.x0, g.nx, hcur.z);
          }
        }
        if (lv == K4) break;
        sync_rows();  // H_lv(qh) complete in every row
        // ----------------------------------------------- E_{lv+1}(q), q = p - lv
        const int qe = qh;
        V3 ecur = {z2, z2, z2};
        if (do_h) {
          const int Q = qe & 1;
          const float* h = LB(2 * lv - 1, Q, r);  // H_lv(qe), row j
          const V3 hc = {hcur.x, hcur.y, hcur.z};
          const float2 hy_im = f2(h[LV - 1], hc.y.x), hz_im = f2(h[2 * LV - 1], hc.z.x);
          const float* hk = LB(2 * lv - 1, Q ^ 1, r);  // H_lv(qe-1), own row
          const V3 eprev = ldv3(LB(2 * lv - 2, Q, r));   // E_lv(qe), own row
          ecur = e_upd2<CAC, CBC>(co, g, i0, j, qe + g.zoff, cdy_e, co.cdz_e[qe], cdx_e, caH[lv], cbH[lv], eprev, hc,
                                  ld2(h - WC), ld2(h + 2 * LV - WC), hy_im, hz_im, ld2(hk), ld2(hk + LV));
          if (src_item) add_src(ecur, lv, qe);
          if (lv + 1 < K4 + 1) stv3(LB(2 * lv, Q, r), ecur);
          if (lv + 1 == K4 && qe >= it.kz0 && qe < it.kz1 && r >= K4 - 1 && r < K4 - 1 + R4 && j < g.ny) {
            const long long gp = gidx(g, i0, j, qe);
            store2(a.out[0], gp, i0, it.x0, g.nx, ecur.x);
            store2(a.out[1], gp, i0, it.x0, g.nx, ecur.y);
            store2(a.out[2], gp, i0, it.x0, g.nx, ecur.z);
          }
        }
        ekp = ecur;  // E_{lv+1}(qe) is the z+1 neighbour of H_{lv+1}(qe-1)
      }
      if (l1) h0p = h0n;
      else h0p = {z2, z2, z2};
    }
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t launch4_t(const FusedArgs& a, const Src4& s, const TMaps& tm, dim3 grid, size_t smem, cudaStream_t st) {
  k_tb4<CAC, CBC, DAC, DBC><<<grid, 32 * (RW4 + 2), smem, st>>>(a, s, tm);
  return cudaGetLastError();
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t limit4_t() {
  return cudaFuncSetAttribute(k_tb4<CAC, CBC, DAC, DBC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

using Launch4Fn = cudaError_t (*)(const FusedArgs&, const Src4&, const TMaps&, dim3, size_t, cudaStream_t);
using Limit4Fn = cudaError_t (*)();
#define YB_B4(m) (m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0
#define YB_T4(m) launch4_t<YB_B4(m)>
#define YB_L4(m) limit4_t<YB_B4(m)>
const Launch4Fn kLaunch4[16] = {YB_T4(0), YB_T4(1), YB_T4(2),  YB_T4(3),  YB_T4(4),  YB_T4(5),  YB_T4(6),  YB_T4(7),
                                YB_T4(8), YB_T4(9), YB_T4(10), YB_T4(11), YB_T4(12), YB_T4(13), YB_T4(14), YB_T4(15)};
const Limit4Fn kLimit4[16] = {YB_L4(0), YB_L4(1), YB_L4(2),  YB_L4(3),  YB_L4(4),  YB_L4(5),  YB_L4(6),  YB_L4(7),
                              YB_L4(8), YB_L4(9), YB_L4(10), YB_L4(11), YB_L4(12), YB_L4(13), YB_L4(14), YB_L4(15)};
#undef YB_B4
#undef YB_T4
#undef YB_L4

}  // namespace

size_t tb4_smem_bytes(int cell_mask, int stages) {
  const int ncoef = (cell_mask & 1) + ((cell_mask >> 1) & 1) + ((cell_mask >> 2) & 1) + ((cell_mask >> 3) & 1);
  const size_t stage = (size_t)(6 * kTB4BY * kTB4Win + ncoef * (kTB4BY - 1) * kTB4Win);
  return (32 + stages * stage + 32 + (size_t)(2 * 4 - 1) * 2 * 3 * kTB4RowWarps * kTB4Win + 32) * 4 +
         (size_t)stages * 16 + 8 * 4;
}

cudaError_t tb4_set_smem_limits() {
  for (int m = 0; m < 16; ++m) {
    const cudaError_t e = kLimit4[m]();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tb4(const FusedArgs& a, const SrcArgs4& s, const TMaps& tm, int cell_mask, dim3 grid,
                       size_t smem, cudaStream_t st) {
  static_assert(sizeof(SrcArgs4) == sizeof(Src4), "source layout");
  return kLaunch4[cell_mask & 15](a, reinterpret_cast<const Src4&>(s), tm, grid, smem, st);
}

}  // namespace yb
