// yb_tb2.cu — temporal blocking of depth 2: TWO full Standard steps per
// sweep (four fused half-steps E1, H1, E2, H2), the GPU analogue of the
// paper's two-step cache-reuse scheme — here the reuse is
// in shared memory instead of a CPU cache, and it halves the HBM bytes per
// cell-update: the state and the per-cell coefficients are read once and the
// state written once per two steps.
//
// Work item = 8 output rows x 128 columns x a z-chunk. The producer warp
// streams the box x0-4..x0+131, y0-2..y0+9 of each read array per plane
// (TMA, mbarrier ring). Per plane p the CTA runs a four-level wavefront:
//   L1  E^{n+1}(p)    rows y0-1..y0+9, cols x0-1..x0+129   -> smem (2 planes)
//   L2  H^{n+3/2}(p-1) rows y0-1..y0+8, cols x0-1..x0+128  -> smem
//   L3  E^{n+2}(p-1)  rows y0..y0+8,   cols x0..x0+128     -> smem (2 planes), rows y0..y0+7 -> HBM
//   L4  H^{n+5/2}(p-2) rows y0..y0+7,   cols x0..x0+127     -> HBM
// (update_e_dof / update_h_dof, kernels.hpp:27-63, PEC folded in, sources at
// steps n and n+1 added after their E level, schedule.hpp:175-199).
// Row warp w owns physical row y0-1+w at every level, so its own-row values
// of earlier planes/levels stay in registers; the x0-1 / x0+128 / x0+129
// columns are computed by a dedicated edge warp (lane = row). One CTA
// barrier per plane (between L2 and L3; the stage is released by per-warp
// arrivals on its "empty" mbarrier). Chunk boundaries re-stream two planes below and one
// above (the wavefront's z-halo). Arithmetic: yee_upd, bit-identical to two
// single steps.
//
// Kernel modes (template MODE): 0 one sweep per launch; 1 + quiescent-item
// skip; 2 several sweeps per launch — items sweep-major, each waits for the
// sweep-(s-1) completion counts of its 3x3-tile x adjacent-chunk neighbourhood
// (every row warp adds 1 to done[item] after a fence; no item-end barrier);
// 3 z-slab peer stores — boundary planes also stored into the neighbours'
// ghost planes, boundary chunks handed out first, in-kernel wait on the
// neighbours' flags and a per-side row-warp count whose last member signals;
// 4 chained exchange periods — 2 and 3 together: several sweeps of one or
// several linked slabs in one launch, per-sweep peer waits and signals
// (FusedArgs::chain; several slabs = the one-GPU emulation of N ranks).
#include <cuda.h>
#include <cuda_runtime.h>

#include "yb_launch.h"
#include "yb_ptx.cuh"

namespace yb {
namespace {

constexpr int RW = kTB2RowWarps;     // 11 row warps: rows y0-1 .. y0+9
constexpr int EDGE = RW;             // warp 11
constexpr int PROD = RW + 1;         // warp 12
constexpr int FACE = RW + 2;         // warp 13
constexpr int BX = kBX;              // 136 smem columns: x = x0-4+c
constexpr int CL = 3, CR = 4 + kTX;  // edge columns x0-1, x0+128 (and CR+1)

constexpr int kConsumers = 32 * (RW + 1);  // row warps + edge warp

// A consumer warp is done reading a stage: every lane's loads have been
// consumed, lane 0 arrives on the stage's "empty" barrier (count RW + 1).
__device__ __forceinline__ void release_stage(uint64_t* empty, int s, int l) {
  __syncwarp();
  if (l == 0) mbar_arrive(smem_u32(&empty[s]));
}

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// true if any source sits on (global-local) plane kl and row j at step bit sb
__device__ __forceinline__ bool src_row(const SrcArgs& s, int sb, int j, int kl) {
  bool hit = false;
  for (int q = 0; q < s.n; ++q) hit |= (s.act[q] & sb) && s.j[q] == j && s.k[q] == kl;
  return hit;
}

struct F4x3 {
  float4 x, y, z;
};

// E update of one float4 group (4 consecutive i) — the same expression as
// the single-step kernel (reference operand order). PEC / non-DoF positions
// are forced to +0 afterwards; the mask pass only runs where some element can
// be masked (boundary tiles, rows, planes), decided warp-uniformly.
template <bool CAC, bool CBC>
__device__ __forceinline__ F4x3 e_update4(const CoefArgs& co, const Geo& g, int i0, bool xedge, int j,
                                          int kg, float cdy, float cdz, float4 cdx, float4 ca,
                                          float4 cb, float4 ex, float4 ey, float4 ez, float4 hx,
                                          float4 hy, float4 hz, float4 hx_jm, float4 hz_jm,
                                          float4 hy_im, float4 hz_im, float4 hx_km, float4 hy_km) {
  F4x3 o;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float A = CAC ? elc(ca, q) : co.ca_s;
    const float B = elc(cb, q);
    el(o.x, q) = yee_upd_t<CAC>(A, elc(ex, q), CBC ? B : cdy, elc(hz, q), elc(hz_jm, q), CBC ? B : cdz,
                         elc(hy, q), elc(hy_km, q));
    el(o.y, q) = yee_upd_t<CAC>(A, elc(ey, q), CBC ? B : cdz, elc(hx, q), elc(hx_km, q),
                         CBC ? B : elc(cdx, q), elc(hz, q), elc(hz_im, q));
    el(o.z, q) = yee_upd_t<CAC>(A, elc(ez, q), CBC ? B : elc(cdx, q), elc(hy, q), elc(hy_im, q),
                         CBC ? B : cdy, elc(hx, q), elc(hx_jm, q));
  }
  const bool kin = kg >= 1 && kg < g.nzg;
  const bool jin = j >= 1 && j < g.ny;
  if (!(jin && kin)) {  // warp-uniform: PEC rows / planes, ghost rows
    const bool jlt = j >= 0 && j < g.ny, kz = kg >= 0 && kg < g.nzg;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q;
      const bool iin = i >= 1 && i < g.nx, ilt = i >= 0 && i < g.nx;
      if (!(ilt && jin && kin)) el(o.x, q) = 0.f;
      if (!(iin && jlt && kin)) el(o.y, q) = 0.f;
      if (!(iin && jin && kz)) el(o.z, q) = 0.f;
    }
  } else if (xedge) {  // the one or two lanes at i = 0 / i >= nx
    if (i0 == 0) {
      o.y.x = 0.f;
      o.z.x = 0.f;
    }
    if (i0 + 4 > g.nx) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q >= g.nx) el(o.x, q) = el(o.y, q) = el(o.z, q) = 0.f;
    }
  }
  return o;
}

// Scalar E update at (i, j, kg).
template <bool CAC, bool CBC>
__device__ __forceinline__ void e_update1(const CoefArgs& co, const Geo& g, int i, int j, int kg,
                                          float cdy, float cdz, float cdx, float ca, float cb,
                                          float ex, float ey, float ez, float hx, float hy, float hz,
                                          float hx_jm, float hz_jm, float hy_im, float hz_im,
                                          float hx_km, float hy_km, float& ox, float& oy, float& oz) {
  const bool kin = kg >= 1 && kg < g.nzg;
  const bool jin = j >= 1 && j < g.ny, jlt = j >= 0 && j < g.ny;
  const bool iin = i >= 1 && i < g.nx, ilt = i >= 0 && i < g.nx;
  const float A = CAC ? ca : co.ca_s;
  ox = (ilt && jin && kin) ? yee_upd_t<CAC>(A, ex, CBC ? cb : cdy, hz, hz_jm, CBC ? cb : cdz, hy, hy_km) : 0.f;
  oy = (iin && jlt && kin) ? yee_upd_t<CAC>(A, ey, CBC ? cb : cdz, hx, hx_km, CBC ? cb : cdx, hz, hz_im) : 0.f;
  oz = (iin && jin && kg >= 0 && kg < g.nzg) ? yee_upd_t<CAC>(A, ez, CBC ? cb : cdx, hy, hy_im, CBC ? cb : cdy, hx, hx_jm)
                                             : 0.f;
}

// Source increments for one E level at global plane kg (step bit `sb`).
__device__ __forceinline__ float src_add(const SrcArgs& s, int sb, int comp, int i, int j, int kl) {
  float v = 0.f;
  bool hit = false;
  for (int q = 0; q < s.n; ++q)
    if ((s.act[q] & sb) && s.comp[q] == comp && s.i[q] == i && s.j[q] == j && s.k[q] == kl) {
      v = sb == 1 ? s.val[q] : s.val2[q];
      hit = true;
    }
  return hit ? v : -0.0f;  // -0 is the additive identity (x + -0 == x for every x)
}

// Per-item geometry shared by the consumer paths.
// pstart..pend: wavefront planes p; pin_end: last plane with input data;
// up: last plane of the H1/E2 levels; pro: a prologue plane (pstart-1, hx/hy).
// Below the global bottom / above the global top there are no planes; inside
// a z-slab the ghost planes -2..-1 and nz..nz+1 stand in for the neighbours.
struct Item {
  int x0, y0, kz0, kz1, pstart, pin_end, pend, up;
  bool pro, src;  // src: some source lies in the item's (halo-extended) box
};

__device__ __forceinline__ Item make_item(const FusedArgs& a, const Geo& g, int item, int T, int ntx) {
  Item it;
  const int chunk = item / T, tile = item - chunk * T;
  it.x0 = (tile % ntx) * kTX;
  it.y0 = (tile / ntx) * kTB2Rows;
  chunk_planes(a, chunk, it.kz0, it.kz1);
  const bool bot = at_bottom(g), top = at_top(g);
  it.pstart = bot ? max(it.kz0 - 1, 0) : it.kz0 - 1;
  it.pro = bot ? it.kz0 >= 2 : true;
  it.pin_end = min(it.kz1 + 1, top ? g.nz - 1 : g.nz + 1);
  it.pend = it.kz1 + 1;
  it.up = min(it.kz1, top ? g.nz - 1 : g.nz);
  it.src = false;
  return it;
}

__device__ __forceinline__ void mark_sources(const SrcArgs& s, Item& it) {
  for (int q = 0; q < s.n; ++q)
    it.src |= s.act[q] != 0 && s.i[q] >= it.x0 - 1 && s.i[q] <= it.x0 + kTX + 1 && s.j[q] >= it.y0 - 1 &&
              s.j[q] <= it.y0 + kTB2Rows + 1 && s.k[q] >= it.pstart && s.k[q] <= it.pend;
}

// Multi-sweep launches: spin (bounded) until every item whose sweep-(sw-1)
// work overlaps this item's reads or writes has published it — the 3 x 3
// tile neighbourhood and the z-chunks covering planes kz0-3 .. kz1+2.
__device__ __noinline__ void wait_neighbours(const FusedArgs& a, int item, int sw) {
  const int T = a.ntx * a.nty, ch = item / T, tile = item - ch * T;
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  int kz0, kz1;
  chunk_planes(a, ch, kz0, kz1);
  const int c_lo = max(kz0 - 3, 0) / a.zchunk, c_hi = min((kz1 + 2) / a.zchunk, a.nch0 - 1);
  const int y_lo = max(ty - 1, 0), y_hi = min(ty + 1, a.nty - 1);
  const int x_lo = max(tx - 1, 0), x_hi = min(tx + 1, a.ntx - 1);
  // every row warp of an item counts itself in done[item] once per sweep
  const unsigned need = (a.epoch + (unsigned)sw) * (unsigned)RW;
  unsigned long long t0 = 0;
  for (long long n = 0;; ++n) {  // one pass of independent relaxed loads, then acquire
    bool ok = true;
    unsigned low = need;  // the smallest count seen (for the error record)
    for (int cc = c_lo; cc <= c_hi; ++cc)
      for (int yy = y_lo; yy <= y_hi; ++yy)
        for (int xx = x_lo; xx <= x_hi; ++xx) {
          unsigned v;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.done + (cc * T + yy * a.ntx + xx)));
          ok &= (int)(v - need) >= 0;
          if ((int)(v - low) < 0) low = v;
        }
    if (ok) break;
    if (n == 0) t0 = globaltimer_ns();
    else if (globaltimer_ns() - t0 > a.wait_ns) {  // report the stuck item instead of hanging
      wait_timed_out(a.err, WAIT_DEP, item, sw, low, need);
      break;
    }
    __nanosleep(128);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Streamed readback order (FusedArgs::diag): work item v of a multi-sweep
// launch -> (sweep, item); sweeps before skew0 sweep-major, the rest along
// y-skewed diagonals d = 2*(sweep - skew0) + tile row, sweeps ascending within
// a diagonal, then z-chunk, then tile column. An item's dependencies (sweep-1,
// tile rows ty-1..ty+1) come earlier (diagonals d-1..d-3, or the sweep-major
// part), so the order is a topological one, and tile row ty finishes its last
// sweep at diagonal 2*(nsweeps-1-skew0) + ty — the bottom rows long before the
// top ones. (Only the last sweeps are skewed: neighbouring tile rows of one
// sweep are a diagonal apart there, so their shared halo rows miss L2.)
__device__ __noinline__ void skew_item(const FusedArgs& a, unsigned long long v, int T, int& sw, int& it) {
  const unsigned long long head = (unsigned long long)a.skewh * a.nitems;
  const unsigned long long flat = (unsigned long long)a.skew0 * a.nitems;
  // Streamed upload: the first skewh sweeps in the mirrored order — position v
  // of the head holds what position head-1-v of a skewed tail holds, with the
  // sweeps and tile rows reversed (a dependency, one sweep later and a row
  // apart in the tail order, becomes one sweep earlier here and still comes
  // first), so tile row 0 of sweep 0 is first and rows follow in ascending order.
  const bool mirror = v < head;
  if (mirror) {
    v = head - 1 - v;
  } else if (v < flat) {
    sw = (int)(v / (unsigned long long)a.nitems);
    it = block_order(a, (int)(v - (unsigned long long)sw * a.nitems), T);
    return;
  } else {
    v -= flat;
  }
  const int per = a.nitems / a.nty;  // items of one (sweep, tile row) group
  const int grp = (int)(v / (unsigned long long)per), rem = (int)(v - (unsigned long long)grp * per);
  const int* dg = mirror ? a.diagh : a.diag;
  int lo = 0, hi = (mirror ? a.ndiagh : a.ndiag) - 1;  // the last diagonal d with dg[d] <= grp
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(dg + mid) <= grp) lo = mid;
    else hi = mid - 1;
  }
  const int sk = max(0, (lo - a.nty + 2) / 2) + (grp - __ldg(dg + lo));
  const int ty = lo - 2 * sk, ch = rem / a.ntx, tx = rem - ch * a.ntx;
  it = ch * T + (mirror ? a.nty - 1 - ty : ty) * a.ntx + tx;
  sw = mirror ? a.skewh - 1 - sk : a.skew0 + sk;
}

// MODE 3 (folded exchange): spin, bounded by the launch's deadline, until a
// neighbour's flag word reaches need.
__device__ __noinline__ void peer_flag_wait(const unsigned* f, unsigned need, int* err, unsigned long long wait_ns,
                                            int item, int side, int code = WAIT_PEER_KERNEL) {
  unsigned long long t0 = 0;
  for (long long n = 0;; ++n) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if ((int)(v - need) >= 0) return;
    if (n == 0) t0 = globaltimer_ns();
    else if (globaltimer_ns() - t0 > wait_ns) {  // the neighbour never signalled
      wait_timed_out(err, code, item, side, v, need);
      return;
    }
    __nanosleep(100);
  }
}

// Stage layout: fields (12 rows from y0-2), then Ca, Cb (11 rows from y0-1),
// then Da, Db (10 rows from y0-1), each present only in per-cell mode.
template <bool CAC, bool CBC, bool DAC, bool DBC>
struct StageLayout {
  static constexpr int floats =
      kTB2Fields + (CAC + CBC) * kTB2SlotC + (DAC + DBC) * kTB2SlotD;
  static constexpr int off_ca = kTB2Fields;
  static constexpr int off_cb = off_ca + CAC * kTB2SlotC;
  static constexpr int off_da = off_cb + CBC * kTB2SlotC;
  static constexpr int off_db = off_da + DAC * kTB2SlotD;
};

struct Bufs {
  float *stages, *e1b, *h1b, *e2b;
  uint64_t *full, *empty;
  __device__ float* E1(int b, int comp, int r, int col) const {
    return e1b + ((size_t)(b * 3 + comp) * RW + r) * BX + col;
  }
  __device__ float* H1(int b, int comp, int r, int col) const {
    return h1b + ((size_t)(b * 3 + comp) * (RW - 1) + r) * BX + col;
  }
  __device__ float* E2(int b, int comp, int r, int col) const {
    return e2b + ((size_t)(b * 3 + comp) * (RW - 2) + r) * BX + col;
  }
  // edge-column state: H0 at CL/CR/CR+1, Da/Db at CL/CR, Ca/Cb at CR
  float* edge;
  __device__ float* H0e(int b, int comp, int r, int e) const { return edge + ((b * 3 + comp) * RW + r) * 3 + e; }
  __device__ float* De(int b, int q, int r, int e) const {
    return edge + 2 * 3 * RW * 3 + ((b * 2 + q) * (RW - 1) + r) * 2 + e;
  }
  __device__ float* Ce(int b, int q, int r) const {
    return edge + 2 * 3 * RW * 3 + 2 * 2 * (RW - 1) * 2 + (b * 2 + q) * RW + r;
  }
};

struct Cursor {
  int s;        // next stage
  uint32_t ph;  // its full-barrier phase parity
  bool peeked;
  __device__ int wait(const Bufs& B, int S) {
    if (!peeked) mbar_wait(smem_u32(&B.full[s]), ph);
    peeked = false;
    const int r = s;
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
    return r;
  }
};

// ============================================================== row warps
// Warp er owns row j = y0-1+er at every level. Carried across planes in
// registers: H0(p-1), Ca/Cb(p-1), Da/Db(p-1), Da/Db(p-2) of its own row;
// E1(p-1) and H1(p-2) of its own row are re-read from shared memory.
// Every shared-memory operand is a per-warp base pointer (selected by the
// plane parity) plus a compile-time offset; the i-1 /
// i+1 neighbours of a lane's float4 are read as one scalar from the row in
// shared memory (column c-1 / c+4; the edge columns for lanes 0 / 31).
template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
struct Rows {
  // MODE: 0 plain, 1 quiescent skip, 2 several sweeps per launch, 3 peer stores,
  // 4 several sweeps with peer stores (chained exchange periods)
  static constexpr bool QS = MODE == 1, MS = MODE == 2 || MODE == 4, PS = MODE == 3 || MODE == 4;
  using L = StageLayout<CAC, CBC, DAC, DBC>;
  static constexpr int E1C = RW * BX, E1B = 3 * E1C;              // comp / buffer strides
  static constexpr int H1C = (RW - 1) * BX, H1B = 3 * H1C;
  static constexpr int E2C = (RW - 2) * BX, E2B = 3 * E2C;

  const FusedArgs& a;
  const Item& it;
  const Bufs& B;
  Cursor& cur;
  float* const* outm;  // this sweep's output buffers (MS)
  const SrcArgs& srcm;  // this sweep's sources (MS)
  const int er, l, j, c, i0;
  const bool xedge;
  const uint64_t st_pol;
  float* const e1o;  // E1 buffer 0, comp 0, row er, column c
  float* const h1o;  // H1 buffer 0, comp 0, row er, column c
  float* const e2o;  // E2 buffer 0, comp 0, row er-1, column c
  float cdy_e, cdy_h;
  float4 cdx_e, cdx_h;
  // cdz values rotate through registers, loaded one plane ahead:
  // ze = cdz_e[p], zh = cdz_h[p-1], ze1 = cdz_e[p-1], zh1 = cdz_h[p-2]
  float ze, zh, ze1, zh1;
  F4x3 h0p;
  float4 cap, cbp, dap, dbp, dap2, dbp2;

  __device__ __forceinline__ Rows(const FusedArgs& a_, const Item& it_, const Bufs& B_, Cursor& cur_,
                                  float* const* out_, const SrcArgs& src_, int er_, int l_, uint64_t pol)
      : a(a_), it(it_), B(B_), cur(cur_), outm(out_), srcm(src_), er(er_), l(l_), j(it_.y0 - 1 + er_), c(4 + 4 * l_),
        i0(it_.x0 + 4 * l_), xedge(i0 == 0 || i0 + 4 > a_.g.nx),
        st_pol(pol),
        e1o(B_.e1b + er_ * BX + c), h1o(B_.h1b + er_ * BX + c), e2o(B_.e2b + (er_ - 1) * BX + c) {
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    cdy_e = a.co.cdy_e[max(j, 0)];
    cdy_h = a.co.cdy_h[max(j, 0)];
    cdx_e = ldg4(a.co.cdx_e + i0);
    cdx_h = ldg4(a.co.cdx_h + i0);
    h0p = {z4, z4, z4};
    cap = cbp = dap = dbp = dap2 = dbp2 = z4;
    ze = a.co.cdz_e[it_.pstart];
    zh = a.co.cdz_h[it_.pstart - 1];
    ze1 = zh1 = 0.f;
  }

  __device__ __forceinline__ float* const* outs() const { return MS ? outm : a.out; }

  __device__ __forceinline__ const SrcArgs& src() const { return MS ? srcm : a.src; }

  __device__ __forceinline__ void prologue() {
    const int rs = er + 1;
    const int s = cur.wait(B, a.nstages);
    const float* F = B.stages + (size_t)s * L::floats + rs * BX + c;
    h0p.x = lds4(F + tb2_fbase(3));
    h0p.y = lds4(F + tb2_fbase(4));
    release_stage(B.empty, s, l);
  }

  // one wavefront plane p (buffers alternate with the plane parity)
  __device__ __forceinline__ void plane(int p) {
    const int PAR = p & 1, Q = PAR ^ 1;  // parity of p, p-1
    const Geo& g = a.g;
    const CoefArgs& co = a.co;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float ze_n = co.cdz_e[p + 1], zh_n = co.cdz_h[p];  // next plane's
    // ------------------------------------------------------- L1: E1(p)
    const bool l1 = p <= it.pin_end;
    F4x3 e1c = {z4, z4, z4}, h0n = {z4, z4, z4};
    float4 can = z4, cbn = z4, dan = z4, dbn = z4;
    int s1 = -1;
    if (l1) {
      s1 = cur.wait(B, a.nstages);
      const float* F = B.stages + (size_t)s1 * L::floats;
      const float* Fr = F + (er + 1) * BX + c;  // field stage row of j
      const float cdz_e = ze;
      h0n.x = lds4(Fr + tb2_fbase(3));
      h0n.y = lds4(Fr + tb2_fbase(4));
      h0n.z = lds4(Fr + tb2_fbase(5));
      const float4 hy_im = make_float4(Fr[tb2_fbase(4) - 1], h0n.y.x, h0n.y.y, h0n.y.z);
      const float4 hz_im = make_float4(Fr[tb2_fbase(5) - 1], h0n.z.x, h0n.z.y, h0n.z.z);
      const float* Fc = F + er * BX + c;  // coefficient stage row of j
      if (CAC) can = lds4(Fc + L::off_ca);
      if (CBC) cbn = lds4(Fc + L::off_cb);
      if (DAC && er <= RW - 2) dan = lds4(Fc + L::off_da);
      if (DBC && er <= RW - 2) dbn = lds4(Fc + L::off_db);
      e1c = e_update4<CAC, CBC>(co, g, i0, xedge, j, p + g.zoff, cdy_e, cdz_e, cdx_e, can, cbn, lds4(Fr + tb2_fbase(0)),
                                lds4(Fr + tb2_fbase(1)), lds4(Fr + tb2_fbase(2)), h0n.x, h0n.y, h0n.z,
                                lds4(Fr + tb2_fbase(3) - BX), lds4(Fr + tb2_fbase(5) - BX), hy_im, hz_im, h0p.x,
                                h0p.y);
      if (it.src && src_row(src(), 1, j, p)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          el(e1c.x, q) = __fadd_rn(el(e1c.x, q), src_add(src(), 1, 0, i0 + q, j, p));
          el(e1c.y, q) = __fadd_rn(el(e1c.y, q), src_add(src(), 1, 1, i0 + q, j, p));
          el(e1c.z, q) = __fadd_rn(el(e1c.z, q), src_add(src(), 1, 2, i0 + q, j, p));
        }
      }
      float* w = e1o + PAR * E1B;
      sts4(w, e1c.x);
      sts4(w + E1C, e1c.y);
      sts4(w + 2 * E1C, e1c.z);
    }
    // No CTA barrier between L1 and L2: L2 reads E1(p-1) (ordered by the
    // previous plane's barrier B) and its own row of E1(p) from registers;
    // the only shared resource L1 frees is the stage.
    if (l1) release_stage(B.empty, s1, l);

    // ----------------------------------------------------- L2: H1(p-1)
    const int kh = p - 1;
    if (kh >= it.pstart && kh <= it.up && er <= RW - 2) {
      const float cdz_h = zh;
      const float* e = e1o + Q * E1B;  // E1(p-1), row j
      const float4 ex_h = lds4(e), ex_jp = lds4(e + BX);
      const float4 ey_h = lds4(e + E1C);
      const float4 ez_h = lds4(e + 2 * E1C), ez_jp = lds4(e + 2 * E1C + BX);
      const float4 ey_ip = make_float4(ey_h.y, ey_h.z, ey_h.w, e[E1C + 4]);
      const float4 ez_ip = make_float4(ez_h.y, ez_h.z, ez_h.w, e[2 * E1C + 4]);
      F4x3 h1c;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float A = DAC ? elc(dap, q) : co.da_s;
        const float Bq = elc(dbp, q);
        el(h1c.x, q) = yee_upd_t<DAC>(A, elc(h0p.x, q), DBC ? Bq : cdz_h, elc(e1c.y, q), elc(ey_h, q),
                                      DBC ? Bq : cdy_h, elc(ez_jp, q), elc(ez_h, q));
        el(h1c.y, q) = yee_upd_t<DAC>(A, elc(h0p.y, q), DBC ? Bq : elc(cdx_h, q), elc(ez_ip, q), elc(ez_h, q),
                                      DBC ? Bq : cdz_h, elc(e1c.x, q), elc(ex_h, q));
        el(h1c.z, q) = yee_upd_t<DAC>(A, elc(h0p.z, q), DBC ? Bq : cdy_h, elc(ex_jp, q), elc(ex_h, q),
                                      DBC ? Bq : elc(cdx_h, q), elc(ey_ip, q), elc(ey_h, q));
      }
      float* w = h1o + Q * H1B;
      sts4(w, h1c.x);
      sts4(w + H1C, h1c.y);
      sts4(w + 2 * H1C, h1c.z);
    }
    consumer_sync();  // (B) H1(p-1) complete

    // ----------------------------------------------------- L3: E2(p-1)
    F4x3 e2c = {z4, z4, z4};
    if (kh >= it.kz0 && kh <= it.up && er >= 1 && er <= RW - 2) {
      const float cdz_e = ze1;
      const float* h = h1o + Q * H1B;    // H1(p-1), row j
      const float* hp = h1o + PAR * H1B;  // H1(p-2), row j
      const float4 hx = lds4(h), hy = lds4(h + H1C), hz = lds4(h + 2 * H1C);
      const float4 hy_im = make_float4(h[H1C - 1], hy.x, hy.y, hy.z);
      const float4 hz_im = make_float4(h[2 * H1C - 1], hz.x, hz.y, hz.z);
      const float* e = e1o + Q * E1B;
      e2c = e_update4<CAC, CBC>(co, g, i0, xedge, j, kh + g.zoff, cdy_e, cdz_e, cdx_e, cap, cbp, lds4(e),
                                lds4(e + E1C), lds4(e + 2 * E1C), hx, hy, hz, lds4(h - BX), lds4(h + 2 * H1C - BX),
                                hy_im, hz_im, lds4(hp), lds4(hp + H1C));
      if (it.src && src_row(src(), 2, j, kh)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          el(e2c.x, q) = __fadd_rn(el(e2c.x, q), src_add(src(), 2, 0, i0 + q, j, kh));
          el(e2c.y, q) = __fadd_rn(el(e2c.y, q), src_add(src(), 2, 1, i0 + q, j, kh));
          el(e2c.z, q) = __fadd_rn(el(e2c.z, q), src_add(src(), 2, 2, i0 + q, j, kh));
        }
      }
      float* w = e2o + Q * E2B;
      sts4(w, e2c.x);
      sts4(w + E2C, e2c.y);
      sts4(w + 2 * E2C, e2c.z);
      const bool own = er <= kTB2Rows && j < g.ny && kh < it.kz1;
      if (own) {  // E^{n+2} of the owned rows -> HBM
        const long long gp = gidx(g, i0, j, kh);
        store_rows3(outs(), gp, i0, g.nx, e2c.x, e2c.y, e2c.z, st_pol);
      }
      if (QS) {
        const bool nz = own && (nonzero4(e2c.x) | nonzero4(e2c.y) | nonzero4(e2c.z));
        if (__any_sync(~0u, nz) && l == 0) qmap_mark(a.qm, (it.y0 / kTB2Rows) * a.ntx + it.x0 / kTX, kh);
      }
    }

    // ----------------------------------------------------- L4: H2(p-2)
    const int k4 = p - 2;
    if (k4 >= it.kz0 && k4 <= it.kz1 - 1 && er >= 1 && er <= kTB2Rows) {
      const float cdz_h = zh1;
      const float* e = e2o + PAR * E2B;  // E2(p-2), row j
      const float4 ex_h = lds4(e), ex_jp = lds4(e + BX);
      const float4 ey_h = lds4(e + E2C);
      const float4 ez_h = lds4(e + 2 * E2C), ez_jp = lds4(e + 2 * E2C + BX);
      const float4 ey_ip = make_float4(ey_h.y, ey_h.z, ey_h.w, e[E2C + 4]);
      const float4 ez_ip = make_float4(ez_h.y, ez_h.z, ez_h.w, e[2 * E2C + 4]);
      const float* h = h1o + PAR * H1B;  // H1(p-2), row j
      const float4 h1x = lds4(h), h1y = lds4(h + H1C), h1z = lds4(h + 2 * H1C);
      F4x3 h2;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float A = DAC ? elc(dap2, q) : co.da_s;
        const float Bq = elc(dbp2, q);
        el(h2.x, q) = yee_upd_t<DAC>(A, elc(h1x, q), DBC ? Bq : cdz_h, elc(e2c.y, q), elc(ey_h, q),
                                     DBC ? Bq : cdy_h, elc(ez_jp, q), elc(ez_h, q));
        el(h2.y, q) = yee_upd_t<DAC>(A, elc(h1y, q), DBC ? Bq : elc(cdx_h, q), elc(ez_ip, q), elc(ez_h, q),
                                     DBC ? Bq : cdz_h, elc(e2c.x, q), elc(ex_h, q));
        el(h2.z, q) = yee_upd_t<DAC>(A, elc(h1z, q), DBC ? Bq : cdy_h, elc(ex_jp, q), elc(ex_h, q),
                                     DBC ? Bq : elc(cdx_h, q), elc(ey_ip, q), elc(ey_h, q));
      }
      if (j < g.ny) {
        const long long gp = gidx(g, i0, j, k4);
        store_rows3(outs() + 3, gp, i0, g.nx, h2.x, h2.y, h2.z, st_pol);
      }
      if (QS && j < g.ny) {
        const bool nz = nonzero4(h2.x) | nonzero4(h2.y) | nonzero4(h2.z);
        if (__any_sync(~0u, nz) && l == 0) qmap_mark(a.qm, (it.y0 / kTB2Rows) * a.ntx + it.x0 / kTX, k4);
      }
    }
    // ---------------------------------------------------------- rotate
    ze1 = ze;
    zh1 = zh;
    ze = ze_n;
    zh = zh_n;
    dap2 = dap;
    dbp2 = dbp;
    if (l1) {
      h0p = h0n;
      cap = can;
      cbp = cbn;
      dap = dan;
      dbp = dbn;
    }
  }
};

template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
__device__ __forceinline__ void tb2_rows(const FusedArgs& a, const Item& it, const Bufs& B, Cursor& cur,
                                         float* const* out, const SrcArgs& src, int er, int l, uint64_t st_pol) {
  Rows<CAC, CBC, DAC, DBC, MODE> R(a, it, B, cur, out, src, er, l, st_pol);
  if (it.pro) R.prologue();
  for (int p = it.pstart; p <= it.pend; ++p) R.plane(p);
}

// Peer stores (MODE 3 / 4), after a boundary item's sweep: row warp er copies
// its own rows (y0..y0+7) of the slab's boundary planes — 0, 1 below, nz-2,
// nz-1 above — of all six next-state components from its own output (just
// written by this thread; read back from L2) into the neighbour's ghost
// planes, over NVLink across GPUs. Outside the plane loop, so the sweep's
// registers are not taxed by the exchange.
__device__ __noinline__ void peer_copy_rows(const FusedArgs& a, const Item& it, float* const* out,
                                            float* const* dn, float* const* up, int er, int l, uint64_t pol) {
  const Geo& g = a.g;
  const int j = it.y0 - 1 + er, i0 = it.x0 + 4 * l;
  if (er < 1 || er > kTB2Rows || j >= g.ny || i0 >= g.nx) return;
  for (int side = 0; side < 2; ++side) {
    float* const* dst = side == 0 ? dn : up;
    if (!dst[0]) continue;
    for (int q = 0; q < 2; ++q) {
      const int k = side == 0 ? q : g.nz - 2 + q;  // my boundary plane
      if (k < it.kz0 || k >= it.kz1) continue;     // not this item's
      const int kp = side == 0 ? a.pdn_k0 + k : k - g.nz;
      const long long src = gidx(g, i0, j, k), dstp = gidx(g, i0, j, kp);
      float4 v[6];
      if (i0 + 3 < g.nx) {
#pragma unroll
        for (int c = 0; c < 6; ++c) v[c] = __ldcg(reinterpret_cast<const float4*>(out[c] + src));
      } else {
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          v[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int e = 0; e < 4; ++e)
            if (i0 + e < g.nx) el(v[c], e) = __ldcg(out[c] + src + e);
        }
      }
      store_rows3(dst, dstp, i0, g.nx, v[0], v[1], v[2], pol);
      store_rows3(dst + 3, dstp, i0, g.nx, v[3], v[4], v[5], pol);
    }
  }
}

// MODE 4, after a boundary item (row warps): each counts itself in its side's
// counter of this sweep once its stores are visible system-wide; the last of
// the side's T * RW row warps publishes psig_val + sweep to the neighbour.
__device__ __noinline__ void chain_signal(const FusedArgs& A, int item, int T, int sw, int nsweeps, int l) {
  const int ch = item / T, nch = A.nitems / T;
  const bool bd = ch == 0 && A.pdn[0], bu = ch == nch - 1 && A.pup[0];
  if (!(bd || bu)) return;
  __syncwarp();
  if (l != 0) return;
  __threadfence_system();
  const unsigned last = (unsigned)T * RW - 1u, val = A.psig_val + (unsigned)sw;
  if (bd && atomicAdd(A.pcnt + sw, 1u) == last) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.psig[0]), "r"(val) : "memory");
  }
  if (bu && atomicAdd(A.pcnt + nsweeps + sw, 1u) == last) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.psig[1]), "r"(val) : "memory");
  }
}

// ============================================================= edge warp
// The columns the row warps' lanes cannot cover: x0-1 (CL), x0+128 (CR),
// x0+129 (CR+1). Work is spread over the lanes as (row, column) tasks per
// level — L1: 11 + 11 + 10 = 32 tasks, L2: 20, L3: 9 — and all state that
// crosses planes (H0, Da/Db, Ca/Cb of these columns) lives in shared memory
// (Bufs::h0e/de/cee), so any lane can pick up any task.
template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
__device__ __forceinline__ void tb2_edge(const FusedArgs& a, const Item& it, const Bufs& B, Cursor& cur,
                                         const SrcArgs& src, int l) {
  using L = StageLayout<CAC, CBC, DAC, DBC>;
  const Geo& g = a.g;
  const CoefArgs& co = a.co;
  const int S = a.nstages;
  // L1 task of this lane: column index e (0: CL, 1: CR, 2: CR+1) and row r
  const int e1i = l < RW ? 0 : (l < 2 * RW ? 1 : 2);
  const int e1r = l - e1i * RW;
  auto ce = [](int e) { return e == 0 ? CL : (e == 1 ? CR : CR + 1); };
  auto ie = [&](int e) { return e == 0 ? it.x0 - 1 : it.x0 + kTX + (e - 1); };
  // L2 task: (column CL|CR, row 0..9) for lanes 0..19
  const int e2i = l < RW - 1 ? 0 : 1, e2r = l - e2i * (RW - 1);
  const bool l2_lane = l < 2 * (RW - 1);
  // L3 task: column CR, rows 1..9 for lanes 0..8
  const int e3r = l + 1;
  const bool l3_lane = l < RW - 2;
  // lane-invariant coefficients of the three tasks
  const int j1 = it.y0 - 1 + e1r, i1 = ie(e1i), j2 = it.y0 - 1 + e2r, i2 = ie(e2i), j3 = it.y0 - 1 + e3r;
  const float cdy1 = co.cdy_e[max(j1, 0)], cdx1 = co.cdx_e[max(i1, 0)];
  const float cdy2 = co.cdy_h[max(j2, 0)], cdx2 = co.cdx_h[max(i2, 0)];
  const float cdy3 = co.cdy_e[max(j3, 0)], cdx3 = co.cdx_e[ie(1)];

  if (it.pro) {  // prologue: H0 hx, hy of plane pstart-1 at the edge columns
    const int s = cur.wait(B, S);
    const float* F = B.stages + (size_t)s * L::floats;
    const int pb = (it.pstart - 1) & 1;
    *B.H0e(pb, 0, e1r, e1i) = F[tb2_fbase(3) + (e1r + 1) * BX + ce(e1i)];
    *B.H0e(pb, 1, e1r, e1i) = F[tb2_fbase(4) + (e1r + 1) * BX + ce(e1i)];
    release_stage(B.empty, s, l);
  }

  for (int p = it.pstart; p <= it.pend; ++p) {
    const bool l1 = p <= it.pin_end;
    if (l1) {
      const int s1 = cur.wait(B, S);
      const float* F = B.stages + (size_t)s1 * L::floats;
      const int r = e1r, col = ce(e1i), i = ie(e1i), j = it.y0 - 1 + r, rs = r + 1;
      const float* Fr = F + rs * BX + col;
      const float hx = Fr[tb2_fbase(3)], hy = Fr[tb2_fbase(4)], hz = Fr[tb2_fbase(5)];
      const float ca = CAC ? F[L::off_ca + r * BX + col] : 0.f;
      const float cb = CBC ? F[L::off_cb + r * BX + col] : 0.f;
      float ox, oy, oz;
      e_update1<CAC, CBC>(co, g, i, j, p + g.zoff, cdy1, co.cdz_e[p], cdx1, ca,
                          cb, Fr[tb2_fbase(0)], Fr[tb2_fbase(1)], Fr[tb2_fbase(2)], hx, hy, hz, Fr[tb2_fbase(3) - BX],
                          Fr[tb2_fbase(5) - BX], Fr[tb2_fbase(4) - 1], Fr[tb2_fbase(5) - 1],
                          *B.H0e((p - 1) & 1, 0, r, e1i), *B.H0e((p - 1) & 1, 1, r, e1i), ox, oy, oz);
      if (it.src && src_row(src, 1, j, p)) {
        ox = __fadd_rn(ox, src_add(src, 1, 0, i, j, p));
        oy = __fadd_rn(oy, src_add(src, 1, 1, i, j, p));
        oz = __fadd_rn(oz, src_add(src, 1, 2, i, j, p));
      }
      *B.E1(p & 1, 0, r, col) = ox;
      *B.E1(p & 1, 1, r, col) = oy;
      *B.E1(p & 1, 2, r, col) = oz;
      *B.H0e(p & 1, 0, r, e1i) = hx;
      *B.H0e(p & 1, 1, r, e1i) = hy;
      *B.H0e(p & 1, 2, r, e1i) = hz;
      if (e1i < 2 && r <= RW - 2) {
        if (DAC) *B.De(p & 1, 0, r, e1i) = F[L::off_da + r * BX + col];
        if (DBC) *B.De(p & 1, 1, r, e1i) = F[L::off_db + r * BX + col];
      }
      if (e1i == 1) {
        *B.Ce(p & 1, 0, r) = ca;
        *B.Ce(p & 1, 1, r) = cb;
      }
      release_stage(B.empty, s1, l);
    }
    __syncwarp();  // L1 lane tasks hand E1 / H0e / De / Ce over to the L2 / L3 lanes

    const int kh = p - 1, hb = kh & 1;
    if (l2_lane && kh >= it.pstart && kh <= it.up) {
      const int r = e2r, col = ce(e2i), i = ie(e2i), j = it.y0 - 1 + r;
      const float A = DAC ? *B.De(hb, 0, r, e2i) : co.da_s;
      const float Bq = DBC ? *B.De(hb, 1, r, e2i) : 0.f;
      const float cdz_h = co.cdz_h[kh], cdy_h = cdy2, cdx = cdx2;
      const float ex_h = *B.E1(hb, 0, r, col), ey_h = *B.E1(hb, 1, r, col), ez_h = *B.E1(hb, 2, r, col);
      // E1(p) at this column (z+1 neighbour); in the top drain plane p = nz
      // it is the PEC zero, not the stale buffer content
      const float exk = l1 ? *B.E1(p & 1, 0, r, col) : 0.f;
      const float eyk = l1 ? *B.E1(p & 1, 1, r, col) : 0.f;
      *B.H1(hb, 0, r, col) = yee_upd_t<DAC>(A, *B.H0e(hb, 0, r, e2i), DBC ? Bq : cdz_h, eyk, ey_h,
                                     DBC ? Bq : cdy_h, *B.E1(hb, 2, r + 1, col), ez_h);
      *B.H1(hb, 1, r, col) = yee_upd_t<DAC>(A, *B.H0e(hb, 1, r, e2i), DBC ? Bq : cdx, *B.E1(hb, 2, r, col + 1), ez_h,
                                     DBC ? Bq : cdz_h, exk, ex_h);
      *B.H1(hb, 2, r, col) = yee_upd_t<DAC>(A, *B.H0e(hb, 2, r, e2i), DBC ? Bq : cdy_h, *B.E1(hb, 0, r + 1, col), ex_h,
                                     DBC ? Bq : cdx, *B.E1(hb, 1, r, col + 1), ey_h);
    }
    consumer_sync();  // (B)

    if (l3_lane && kh >= it.kz0 && kh <= it.up) {
      const int r = e3r, i = ie(1), j = it.y0 - 1 + r;
      float ox, oy, oz;
      e_update1<CAC, CBC>(co, g, i, j, kh + g.zoff, cdy3, co.cdz_e[kh], cdx3,
                          *B.Ce(hb, 0, r), *B.Ce(hb, 1, r), *B.E1(hb, 0, r, CR), *B.E1(hb, 1, r, CR),
                          *B.E1(hb, 2, r, CR), *B.H1(hb, 0, r, CR), *B.H1(hb, 1, r, CR), *B.H1(hb, 2, r, CR),
                          *B.H1(hb, 0, r - 1, CR), *B.H1(hb, 2, r - 1, CR), *B.H1(hb, 1, r, CR - 1),
                          *B.H1(hb, 2, r, CR - 1), *B.H1(hb ^ 1, 0, r, CR), *B.H1(hb ^ 1, 1, r, CR), ox, oy,
                          oz);
      if (it.src && src_row(src, 2, j, kh)) {
        ox = __fadd_rn(ox, src_add(src, 2, 0, i, j, kh));
        oy = __fadd_rn(oy, src_add(src, 2, 1, i, j, kh));
        oz = __fadd_rn(oz, src_add(src, 2, 2, i, j, kh));
      }
      *B.E2(hb, 0, r - 1, CR) = ox;
      *B.E2(hb, 1, r - 1, CR) = oy;
      *B.E2(hb, 2, r - 1, CR) = oz;
    }
    // lanes read other lanes' E1/Ce slots in L3 that the next L1 rewrites
    __syncwarp();
  }
}

// The kernel body. MODE 4 with CHP: several slabs, `chain` points at their
// arguments in parameter space (ChainParams) and every per-item field access
// is a constant-bank load with a register offset; without CHP (one slab, a
// rank's launch) `a` is the slab itself and its fields stay immediate
// constant operands, as in the other modes.
template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE, bool CHP>
__device__ __forceinline__ void tb2_body(const FusedArgs& a, const TMaps& tm, const TMaps& tm_o,
                                         const ChainSlab* chain) {
  constexpr bool QS = MODE == 1, MS = MODE == 2 || MODE == 4, PS = MODE == 3 || MODE == 4, CH = MODE == 4;
  using L = StageLayout<CAC, CBC, DAC, DBC>;
  constexpr int NARR = 6 + CAC + CBC + DAC + DBC;
  constexpr uint32_t kBytesF = kBX * kTB2BY * 4, kBytesE = kBX * kTB2RowsE * 4, kBytesC = kBX * kTB2RowsCA * 4,
                     kBytesD = kBX * kTB2RowsDA * 4;
  constexpr uint32_t kStageBytes = 2 * kBytesF + 4 * kBytesE + (CAC + CBC) * kBytesC + (DAC + DBC) * kBytesD;
  constexpr int kQ = 8;
  extern __shared__ __align__(128) float smem[];

  const Geo& g = a.g;
  const CoefArgs& co = a.co;
  const int S = a.nstages;
  Bufs B;
  B.stages = smem;
  B.e1b = smem + (size_t)S * L::floats;
  B.h1b = B.e1b + kTB2E1;
  B.e2b = B.h1b + kTB2H1;
  B.edge = B.e2b + kTB2E2;
  B.full = reinterpret_cast<uint64_t*>(B.edge + kTB2Edge);
  B.empty = B.full + S;
  int* item_q = reinterpret_cast<int*>(B.empty + S);
  int* sweep_q = item_q + kQ;
  int* slab_q = sweep_q + kQ;  // MODE 4: the item's slab in a.chain
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int T = a.ntx * a.nty;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&B.full[s]), 1);
      mbar_init(smem_u32(&B.empty[s]), RW + 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (w == FACE) {  // upper-face DoFs, two steps per sweep: h <- Da*(Da*h + 0) + 0
    // (no sweep reads them for a valid update, so all sweeps' steps are applied
    // here in order, into the buffer that holds the launch's final state)
    if (a.no_faces) return;
    if (CH) {  // every slab of the chain, all sweeps in order, into its final-state buffer
      for (int sl = 0; sl < a.nchain; ++sl) {
        const FusedArgs& A = CHP ? chain[sl].a : a;
        const long long nf = face_points(A.g);
        float* const* fin =
            (a.nsweeps & 1) ? A.out : const_cast<float* const*>(reinterpret_cast<const float* const*>(A.in));
        for (long long t = blockIdx.x * 32LL + l; t < nf; t += gridDim.x * 32LL) {
          face_point(A.g, A.in, fin, A.co, t);
          for (int q = 1; q < 2 * a.nsweeps; ++q) face_point(A.g, fin, fin, A.co, t);
        }
      }
      return;
    }
    const long long nf = face_points(g);
    if (!MS) {
      for (long long t = blockIdx.x * 32LL + l; t < nf; t += gridDim.x * 32LL) {
        face_point(g, a.in, a.out, co, t);
        face_point(g, a.out, a.out, co, t);
      }
      return;
    }
    float* const* fin = (a.nsweeps & 1) ? a.out : const_cast<float* const*>(reinterpret_cast<const float* const*>(a.in));
    if (MODE == 2 && a.upband) {  // streamed upload: the face DoFs span every tile row
      if (l == 0) peer_flag_wait(a.upband + a.nty - 1, a.up_need, a.err, a.wait_ns, -1, a.nty - 1, WAIT_UPLOAD);
      __syncwarp();
    }
    for (long long t = blockIdx.x * 32LL + l; t < nf; t += gridDim.x * 32LL) {
      face_point(g, a.in, fin, co, t);
      for (int q = 1; q < 2 * a.nsweeps; ++q) face_point(g, fin, fin, co, t);
    }
    if (MODE == 2 && a.band) {  // streamed readback: this CTA's face DoFs are final
      __syncwarp();
      if (l == 0) {
        __threadfence_system();
        atomicAdd(a.band + a.nty, 1u);
      }
    }
    return;
  }

  if (w == PROD) {  // TMA producer (one lane)
    if (l != 0) return;
    int p_item = -1, p_e = 0, p_nE = 0, p_seq = 0, p_sweep = 0, p_slab = 0;
    for (int q = 0;; ++q) {
      const int s = q % S;
      if (q >= S) mbar_wait(smem_u32(&B.empty[s]), (uint32_t)(((q / S) - 1) & 1));
      const uint32_t bar = smem_u32(&B.full[s]);
      if (p_item < 0) {
        const unsigned long long v = atomicAdd(a.sched, 1ull) - a.sched_base;
        int it = -1, sw = 0, sl = 0;
        if (CH) {  // (sweep, slab, item) in z order: the chunks of all slabs, bottom to top, per sweep
          // (not MODE 3's boundary-chunks-first order: with several sweeps in flight that
          // would make each sweep's top chunk wait for the previous sweep's last chunk)
          const unsigned long long tot = (unsigned long long)a.chain_off[a.nchain];
          if (v < tot * a.nsweeps) {
            sw = (int)(v / tot);
            const int r = (int)(v - (unsigned long long)sw * tot);
            while (sl + 1 < a.nchain && r >= a.chain_off[sl + 1]) ++sl;
            it = block_order(a, r - a.chain_off[sl], T);  // within a chunk: column blocks, as MODE 2
          }
        } else if (!MS) {
          it = v < (unsigned long long)a.nitems ? (int)v : -1;
          if (PS && it >= 0 && a.pfold) {  // bottom chunk, top chunk, then the interior
            const int nch = a.nitems / T, q = it / T, tile = it - q * T;
            const int ch = a.pfold == 2 ? q : (q == 0 ? 0 : (q == 1 ? nch - 1 : q - 1));
            it = ch * T + tile;
            const bool wd = ch == 0 && a.pdn[0], wu = ch == nch - 1 && a.pup[0];
            if (wd) peer_flag_wait(a.pflag, a.pneed, a.perr, a.wait_ns, it, 0);
            if (wu) peer_flag_wait(a.pflag + 1, a.pneed, a.perr, a.wait_ns, it, 1);
            if (wd || wu) asm volatile("fence.proxy.async.global;" ::: "memory");  // their stores, then our TMA reads
          }
        } else if (v < (unsigned long long)a.nitems * a.nsweeps) {
          if (MODE == 2 && a.diag) {
            skew_item(a, v, T, sw, it);
          } else {
            sw = (int)(v / (unsigned long long)a.nitems);
            it = (int)(v - (unsigned long long)sw * a.nitems);
            if (MODE == 2) it = block_order(a, it, T);
          }
        }
        item_q[p_seq % kQ] = it;
        if (MS) sweep_q[p_seq % kQ] = sw;
        if (CH) slab_q[p_seq % kQ] = sl;
        ++p_seq;
        if (it < 0) {
          mbar_arrive(bar);
          return;
        }
        const FusedArgs& A = CHP ? chain[sl].a : a;
        if (MODE == 2 && a.upband && sw == 0) {  // streamed upload: my tile rows (and the halo rows above) have landed
          const int q = min((it % T) / a.ntx + 1, a.nty - 1);
          peer_flag_wait(a.upband + q, a.up_need, a.err, a.wait_ns, it, q, WAIT_UPLOAD);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the copy engine's writes, then our TMA reads
        }
        if (MS && sw > 0) {  // the neighbourhood must have finished the previous sweep
          wait_neighbours(A, it, sw);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // their stores, then our TMA reads
        }
        if (CH) {  // a boundary item: the neighbour's sweep sw-1 has stored my ghost planes
          const int nch = A.nitems / T, ch = it / T;
          const bool wd = ch == 0 && A.pdn[0], wu = ch == nch - 1 && A.pup[0];
          if (wd) peer_flag_wait(A.pflag, A.pneed + (unsigned)sw, A.perr, A.wait_ns, it, 0);
          if (wu) peer_flag_wait(A.pflag + 1, A.pneed + (unsigned)sw, A.perr, A.wait_ns, it, 1);
          if (wd || wu) asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        p_sweep = sw;
        p_slab = sl;
#ifdef YB_TB2_STAMP
        if (MODE == 2 && a.stamp) a.stamp[2 * ((size_t)sw * a.nitems + it)] = globaltimer_ns();
#endif
        const Item pi = make_item(A, A.g, it, T, a.ntx);
        if (QS) {  // quiescent item: input box all +0, no source in either step -> skip
          const int tl = it % T;
          const int k0 = pi.pro ? pi.pstart - 1 : pi.pstart;
          if (!src_in_box(a.src, pi.x0 - 4, pi.x0 + kTX + 3, pi.y0 - 2, pi.y0 + kTB2Rows + 1, k0, pi.pin_end) &&
              !qmap_dirty(a.qm, tl % a.ntx, tl / a.ntx, k0, pi.pin_end)) {
            item_q[(p_seq - 1) % kQ] = it | kSkipItem;
            atomicAdd(a.skipped, 1ull);
            mbar_arrive(bar);
            continue;  // the item occupies this one (empty) stage
          }
        }
        p_item = it;
        p_e = 0;
        p_nE = (pi.pro ? 1 : 0) + pi.pin_end - pi.pstart + 1;
      }
      const FusedArgs& PA = CHP ? chain[p_slab].a : a;
      const Item pi = make_item(PA, PA.g, p_item, T, a.ntx);
      const int x0 = pi.x0, y0 = pi.y0;
      const int pro = pi.pro ? 1 : 0;
      const TMaps& M = CHP ? ((p_sweep & 1) ? chain[p_slab].tm_o : chain[p_slab].tm)
                           : ((MS && (p_sweep & 1)) ? tm_o : tm);  // this sweep's input state
      float* dst = B.stages + (size_t)s * L::floats;
      // tensor z coordinate = local plane + kGhost
      if (pro && p_e == 0) {  // hx, hy of plane pstart-1
        mbar_expect_tx(bar, kBytesF + kBytesE);
        tma_load_3d(smem_u32(dst + tb2_foff(3)), &M.m[3], x0 - 4, y0 - 2, pi.pstart - 1 + kGhost, bar);
        tma_load_3d(smem_u32(dst + tb2_foff(4)), &M.m[4], x0 - 4, y0 - 1, pi.pstart - 1 + kGhost, bar);
      } else {
        const int z = pi.pstart + p_e - pro + kGhost;
        mbar_expect_tx(bar, kStageBytes);
#pragma unroll
        for (int q2 = 0; q2 < 6; ++q2)
          tma_load_3d(smem_u32(dst + tb2_foff(q2)), &M.m[q2], x0 - 4, tb2_short(q2) ? y0 - 1 : y0 - 2, z, bar);
        int m = 6;
        if (CAC) tma_load_3d(smem_u32(dst + L::off_ca), &M.m[m++], x0 - 4, y0 - 1, z, bar);
        if (CBC) tma_load_3d(smem_u32(dst + L::off_cb), &M.m[m++], x0 - 4, y0 - 1, z, bar);
        if (DAC) tma_load_3d(smem_u32(dst + L::off_da), &M.m[m++], x0 - 4, y0 - 1, z, bar);
        if (DBC) tma_load_3d(smem_u32(dst + L::off_db), &M.m[m++], x0 - 4, y0 - 1, z, bar);
        (void)NARR;
        // the same boxes a.pf planes further on, into L2 only (within the item's planes)
        if (a.pf > 0 && z + a.pf <= pi.pin_end + kGhost) {
#pragma unroll
          for (int q2 = 0; q2 < 6; ++q2)
            tma_prefetch_3d(&M.m[q2], x0 - 4, tb2_short(q2) ? y0 - 1 : y0 - 2, z + a.pf);
#pragma unroll
          for (int q2 = 6; q2 < NARR; ++q2) tma_prefetch_3d(&M.m[q2], x0 - 4, y0 - 1, z + a.pf);
        }
      }
#ifdef YB_TB2_STAMP
      if (MODE == 2 && a.stamp && p_e + 1 == p_nE) a.stamp[2 * ((size_t)p_sweep * a.nitems + p_item) + 1] = globaltimer_ns();
#endif
      if (++p_e == p_nE) p_item = -1;
    }
  }

  uint64_t st_pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(st_pol));
  Cursor cur{0, 0u, false};
  int c_seq = 0;
  for (;;) {
    mbar_wait(smem_u32(&B.full[cur.s]), cur.ph);
    cur.peeked = true;
    const int item = item_q[c_seq % kQ];
    const int sw = MS ? sweep_q[c_seq % kQ] : 0;
    const FusedArgs& A = CHP ? chain[slab_q[c_seq % kQ]].a : a;
    ++c_seq;
    if (item < 0) break;
    if (QS && (item & kSkipItem)) {  // quiescent: consume the empty stage, nothing to write
      release_stage(B.empty, cur.wait(B, S), l);
      continue;
    }
    const SrcArgs& src = MS ? A.srcs[sw] : A.src;
    float* const* out = (MS && (sw & 1)) ? const_cast<float* const*>(reinterpret_cast<const float* const*>(A.in)) : A.out;
    Item it = make_item(A, A.g, item, T, a.ntx);
    mark_sources(src, it);
    if (w == EDGE)
      tb2_edge<CAC, CBC, DAC, DBC, MODE>(A, it, B, cur, src, l);
    else
      tb2_rows<CAC, CBC, DAC, DBC, MODE>(A, it, B, cur, out, src, w, l, st_pol);
    if (PS && w < RW) {  // an item's rows of the slab's boundary planes -> the neighbours' ghost planes
      // (by plane, not by chunk: unfolded MODE 3 launches may cut 1-plane chunks)
      if ((it.kz0 < 2 && A.pdn[0]) || (it.kz1 > A.g.nz - 2 && A.pup[0])) {
        const bool odd = CH && (sw & 1);  // MODE 4: the neighbours' buffers of this sweep's output parity
        peer_copy_rows(A, it, out, odd ? A.pdn_o : A.pdn, odd ? A.pup_o : A.pup, w, l, st_pol);
      }
    }
    if (CH) {  // boundary item: per sweep and side, the last row warp signals the neighbour
      if (w < RW) chain_signal(A, item, T, sw, a.nsweeps, l);
    } else if (PS) {  // boundary item: its peer stores before the signal
      const int ch = item / T, nch = a.nitems / T;
      const bool bd = ch == 0 && a.pdn[0], bu = ch == nch - 1 && a.pup[0];
      if (bd || bu) {
        if (!a.pfold) {
          __threadfence_system();  // before the separate signal launch
        } else if (w < RW) {
          // each row warp counts itself once its stores are visible system-wide
          // (its peer stores; every stage it consumed — the ghost planes read —
          // had landed); the last of the T * RW row warps of the side signals
          __syncwarp();
          if (l == 0) {
            __threadfence_system();
            const unsigned last = (unsigned)T * RW - 1u;
            if (bd && atomicAdd(a.pcnt, 1u) - a.pcnt_base[0] == last) {
              __threadfence_system();
              asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.psig[0]), "r"(a.psig_val) : "memory");
            }
            if (bu && atomicAdd(a.pcnt + 1, 1u) - a.pcnt_base[1] == last) {
              __threadfence_system();
              asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.psig[1]), "r"(a.psig_val) : "memory");
            }
          }
        }
      }
    }
    if (MS && w < RW) {  // publish: this row warp's part of sweep sw is in global memory
      __syncwarp();
      if (l == 0) {
        __threadfence();
        atomicAdd(A.done + item, 1u);
        if (MODE == 2 && A.band && sw == a.nsweeps - 1) {  // streamed readback: my rows of the band are final
          __threadfence_system();
          atomicAdd(A.band + (item % T) / a.ntx, 1u);
        }
      }
    }
  }
}

template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
__global__ void __maxnreg__(128) k_tb2(const __grid_constant__ FusedArgs a, const __grid_constant__ TMaps tm,
                                       const __grid_constant__ TMaps tm_o) {
  tb2_body<CAC, CBC, DAC, DBC, MODE, false>(a, tm, tm_o, nullptr);
}

// MODE 4: the launch's schedule arguments and every slab's arguments and read
// maps as kernel parameters (8 x 3.5 KB + 0.9 KB, within the 32 KB limit)
struct ChainParams {
  FusedArgs a;
  ChainSlab s[kChainMax];
};

template <bool CAC, bool CBC, bool DAC, bool DBC>
__global__ void __maxnreg__(128) k_tb2_chain(const __grid_constant__ ChainParams P) {
  tb2_body<CAC, CBC, DAC, DBC, 4, true>(P.a, P.s[0].tm, P.s[0].tm_o, P.s);
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t launch_chain_t(const ChainParams& P, dim3 grid, size_t smem, cudaStream_t st) {
  k_tb2_chain<CAC, CBC, DAC, DBC><<<grid, kTB2Threads, smem, st>>>(P);
  return cudaGetLastError();
}

template <bool CAC, bool CBC, bool DAC, bool DBC>
cudaError_t set_limit_chain_t() {
  return cudaFuncSetAttribute(k_tb2_chain<CAC, CBC, DAC, DBC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024);
}

template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
cudaError_t launch_t(const FusedArgs& a, const TMaps& tm, const TMaps& tm_o, dim3 grid, size_t smem,
                     cudaStream_t st) {
  k_tb2<CAC, CBC, DAC, DBC, MODE><<<grid, kTB2Threads, smem, st>>>(a, tm, tm_o);
  return cudaGetLastError();
}

template <bool CAC, bool CBC, bool DAC, bool DBC, int MODE>
cudaError_t set_limit_t() {
  return cudaFuncSetAttribute(k_tb2<CAC, CBC, DAC, DBC, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024);
}

using LaunchFn = cudaError_t (*)(const FusedArgs&, const TMaps&, const TMaps&, dim3, size_t, cudaStream_t);
using LimitFn = cudaError_t (*)();

// index: bits 0-3 per-cell Ca/Cb/Da/Db, then 16 * MODE (0..4)
#define YB_B(m) (m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0, (m >> 4)
#ifdef YB_TB2_AB  // measurement builds (tools/ab_build.sh): only the multi-sweep kernels of configs 1 / 2, 4 / 3, 5
template <int M>
constexpr bool ab_has = (M >> 4) == 2 && ((M & 15) == 0 || (M & 15) == 2 || (M & 15) == 15);
template <int M>
cudaError_t ab_launch(const FusedArgs& a, const TMaps& tm, const TMaps& tm_o, dim3 grid, size_t smem, cudaStream_t st) {
  if constexpr (ab_has<M>) return launch_t<YB_B(M)>(a, tm, tm_o, grid, smem, st);
  return cudaErrorNotSupported;
}
template <int M>
cudaError_t ab_limit() {
  if constexpr (ab_has<M>) return set_limit_t<YB_B(M)>();
  return cudaSuccess;
}
#define YB_T(m) ab_launch<m>
#define YB_L(m) ab_limit<m>
#else
#define YB_T(m) launch_t<YB_B(m)>
#define YB_L(m) set_limit_t<YB_B(m)>
#endif
#define YB_8(F, b) F(b), F(b + 1), F(b + 2), F(b + 3), F(b + 4), F(b + 5), F(b + 6), F(b + 7)
const LaunchFn kLaunch[80] = {YB_8(YB_T, 0),  YB_8(YB_T, 8),  YB_8(YB_T, 16), YB_8(YB_T, 24),
                              YB_8(YB_T, 32), YB_8(YB_T, 40), YB_8(YB_T, 48), YB_8(YB_T, 56),
                              YB_8(YB_T, 64), YB_8(YB_T, 72)};
const LimitFn kLimit[80] = {YB_8(YB_L, 0),  YB_8(YB_L, 8),  YB_8(YB_L, 16), YB_8(YB_L, 24),
                            YB_8(YB_L, 32), YB_8(YB_L, 40), YB_8(YB_L, 48), YB_8(YB_L, 56),
                            YB_8(YB_L, 64), YB_8(YB_L, 72)};
using ChainFn = cudaError_t (*)(const ChainParams&, dim3, size_t, cudaStream_t);
#ifdef YB_TB2_AB
inline cudaError_t ab_chain(const ChainParams&, dim3, size_t, cudaStream_t) { return cudaErrorNotSupported; }
inline cudaError_t ab_chain_limit() { return cudaSuccess; }
#define YB_C(m) ab_chain
#define YB_CL(m) ab_chain_limit
#else
#define YB_C(m) launch_chain_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0>
#define YB_CL(m) set_limit_chain_t<(m & 1) != 0, (m & 2) != 0, (m & 4) != 0, (m & 8) != 0>
#endif
const ChainFn kChain[16] = {YB_8(YB_C, 0), YB_8(YB_C, 8)};
const LimitFn kChainLimit[16] = {YB_8(YB_CL, 0), YB_8(YB_CL, 8)};
#undef YB_C
#undef YB_CL
#undef YB_8
#undef YB_T
#undef YB_L
#undef YB_B

}  // namespace

cudaError_t tb2_set_smem_limits() {
  for (int m = 0; m < 80; ++m) {
    const cudaError_t e = kLimit[m]();
    if (e != cudaSuccess) return e;
  }
  for (int m = 0; m < 16; ++m) {
    const cudaError_t e = kChainLimit[m]();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tb2(const FusedArgs& a, const TMaps& tm, const TMaps& tm_out, int cell_mask, dim3 grid,
                       size_t smem, cudaStream_t st) {
  const int mode = a.nchain > 0 ? 4 : (a.pdn[0] || a.pup[0]) ? 3 : (a.nsweeps > 1 ? 2 : (a.qm.bits ? 1 : 0));
  return kLaunch[(cell_mask & 15) | (mode << 4)](a, tm, tm_out, grid, smem, st);
}

cudaError_t launch_tb2_chain(const FusedArgs& a, const ChainSlab* slabs, int n, int cell_mask, dim3 grid,
                             size_t smem, cudaStream_t st) {
  if (n < 1 || n > kChainMax) return cudaErrorInvalidValue;
  thread_local ChainParams P;  // ~29 KB: not on the stack
  P.a = a;
  P.a.nchain = n;
  for (int i = 0; i < n; ++i) P.s[i] = slabs[i];
  return kChain[cell_mask & 15](P, grid, smem, st);
}

}  // namespace yb
