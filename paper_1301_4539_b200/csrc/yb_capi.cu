// yb_capi.cu — the C-ABI of libyeeb200.so (include/yeeb200.h): device-resident
// padded SoA state, coefficient management, TMA descriptor setup and the
// Standard-step time loop. Host side of the B200 path; no CPU compute path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/yeeb200.h"
#include "../../include/yeeb200_inputs.h"
#include "yb_launch.h"

using yb::Geo;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define YB_CU(expr)                                                                       \
  do {                                                                                    \
    const cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                                \
      return fail(YB_CUDA_ERROR, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                              \
  } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

struct Src {
  int comp, i, j, k;
  std::vector<float> table;
};

struct Probe {
  int comp, i, j, k, stride;
};

// A neighbouring slab reachable through peer memory (same process, or a
// CUDA IPC mapping of another process's allocations).
struct PeerSide {
  bool on = false;
  float* buf[2][6] = {};      // its state buffers (plane 0 pointers)
  unsigned* flags = nullptr;  // its flag words: [0] written by its lower neighbour, [1] by its upper
  int nz = 0;
  std::vector<void*> ipc;  // IPC mappings to close
};

struct TimerPair {
  cudaEvent_t a, b;
};

int comp_ext(const Geo& g, int c, int e[3]) {
  const int n[3] = {g.nx, g.ny, g.nz};
  const int axis = c % 3;
  for (int a = 0; a < 3; ++a) {
    const bool node = c < 3 ? (a != axis) : (a == axis);
    e[a] = n[a] + (node ? 1 : 0);
  }
  return 0;
}

}  // namespace

struct yb_sim {
  Geo g{};
  int device = 0, variant = YB_VARIANT_FUSED, zchunk_req = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  float* buf[2][6] = {};
  int cur = 0;
  float* cell[4] = {};  // per-cell arrays (nullptr = uniform / axis)
  float ca_s = 1.0f, da_s = 1.0f;
  bool cb_uniform = false, db_uniform = false;
  float cb_u = 0.f, db_u = 0.f;
  std::vector<float> axis_ref[3];  // reference per-axis coefficients (host copy)
  float* axis_dev[6] = {};         // cdx_e, cdy_e, cdz_e, cdx_h, cdy_h, cdz_h
  int axis_len[3] = {};
  std::vector<Src> sources;
  int64_t step_index = 0, steps = 0, launches = 0;
  yb::TMaps tm[2];
  bool tm_valid = false;
  bool timing = false;
  std::vector<TimerPair> timers;
  size_t timers_used = 0;
  double kernel_ms = 0.0;
  int64_t kernel_timed = 0;
  size_t dev_bytes = 0;
  int stages = 0;
  dim3 grid{1, 1, 1};
  int zchunk = 0;
  int ntx = 1, nty = 1, nitems = 1;
  yb::TMaps tm2[2];  // two-step sweep maps (taller boxes)
  int stages2 = 0, zchunk2 = 0, nitems2 = 1;
  int zchunk2p = 0;  // z-chunk of multi-sweep launches (0: this grid does not use them)
  dim3 grid2{1, 1, 1};
  yb::TMaps tm4[2];  // four-step sweep maps (64-column window boxes)
  unsigned* done = nullptr;   // multi-sweep launches: per-item completion epochs
  int done_n = 0;
  unsigned epoch = 0;
  yb::SrcArgs* srcs_dev = nullptr;  // per-sweep sources of a multi-sweep launch
  int srcs_cap = 0;
  int stages4 = 0, zchunk4 = 0, ntx4 = 1, nty4 = 1;
  unsigned long long* sched = nullptr;  // device work counter of the fused kernel
  unsigned long long sched_base = 0;
  std::vector<Probe> probes;
  float* probe_dev = nullptr;  // recorded values (device)
  size_t probe_cap = 0;        // capacity of probe_dev (floats)
  std::vector<std::pair<int64_t, int>> probe_meta;  // (step, probe) per recorded value
  float* snap_h[3] = {};        // HSnapshot (planes 0..nz of hx, hy, hz)
  bool have_snap = false;
  double* energy_dev = nullptr;  // weights | partials | result
  int store_policy = 1;  // evict_first (YB_STPOL overrides; tuning knob)
  int pending = 0;            // steps of a split sweep in flight (yb_advance_begin)
  // split sweeps: the interior launch runs on a side stream with its own
  // work counter, concurrently with the boundary launch and the exchange
  cudaStream_t side = nullptr;
  cudaStream_t xfer = nullptr;  // layout conversion of yb_upload_fields / yb_download_fields
  cudaEvent_t xev[7] = {};
  cudaEvent_t ev_pre = nullptr, ev_int = nullptr;
  unsigned long long* sched2 = nullptr;
  unsigned long long sched2_base = 0;
  bool on_side = false;
  PeerSide peer[2];           // direct halo push targets (0: below, 1: above)
  unsigned* pflags = nullptr; // my flag words [0] from below, [1] from above, [2] error
  int* cflags = nullptr;      // uniformity flags of yb_set_cell_coeffs_n
  unsigned push_count = 0;
  cudaStream_t peer_stream = nullptr;
  cudaEvent_t peer_go = nullptr, peer_done = nullptr;
  bool peer_inflight = false;
  bool peer_stores = false;   // the next two-step launch also writes the neighbours' ghost planes
  bool peer_folded = false;   // ... and did its own wait / signal (set by step_tb2)
  unsigned pcnt_base[2] = {0u, 0u};
  bool pending_full = false;  // ... whose boundary launch already covered every plane
  bool persist = true;        // multi-sweep two-step launches (YB_TB2_PERSIST=0: off)
  int pf2 = 0;                // two-step L2 prefetch distance in planes (YB_TB2_PF)
  int xblock = 4;             // multi-sweep item order: column blocks of this many tiles (YB_TB2_XBLOCK; 0: row-major)
  bool qskip = false;         // yb_set_quiescent_skip
  bool q_valid = false;       // quiescent map matches the state buffers
  unsigned* qbits = nullptr;  // quiescent map (tiles x words)
  int qwords = 0, qtiles = 0;
  unsigned long long* qskipped = nullptr;  // device counter of skipped items
  int* werr = nullptr;        // wait-error record of the bounded spin waits (yb::WaitErr, 8 ints)
  unsigned long long wait_ns = 20000000000ull;  // their deadline (YB_WAIT_TIMEOUT_MS, default 20 s)
  // chained exchange periods (yb_peer_run, two-step kernel MODE 4)
  unsigned* pcnt4 = nullptr;            // per side and sweep: boundary row warps done (2 x kChainSweeps)
  cudaEvent_t chain_ev = nullptr;
  // streamed readback (yb_run_to_host): skewed item order of the last launch,
  // per tile-row completion counters (+ faces) polled by the copy stream
  bool drain = false;         // the next multi-sweep launch skews its last sweeps and counts bands
  int* diag_dev = nullptr;    // diagonal offsets (FusedArgs::diag)
  int diag_cap = 0, diag_sweeps = 0, diag_nty = 0, ndiag = 0;
  unsigned* band_dev = nullptr;  // nty tile-row counters + 1 face counter (monotonic)
  int band_n = 0;
  unsigned band_base = 0, face_base = 0;
  unsigned last_grid = 0;     // CTAs of the last two-step launch
  int64_t streamed = 0;       // yb_run_to_host calls that streamed
  // streamed upload (yb_run_streamed): the first sweeps of the launch follow the host->device
  // copies tile row by tile row (per-row words written by the copy stream)
  bool upstream = false;      // the next multi-sweep launch skews its first sweeps and waits on upband
  int* diagh_dev = nullptr;   // diagonal offsets of the head skew (FusedArgs::diagh)
  int diagh_cap = 0, diagh_sweeps = 0, diagh_nty = 0, ndiagh = 0;
  unsigned* upband_dev = nullptr;  // nty words (monotonic)
  int upband_n = 0;
  unsigned up_base = 0;
  int64_t streamed_up = 0;    // yb_run_streamed calls whose upload overlapped the run
};

namespace {

int cell_mask(const yb_sim* s) {
  int m = 0;
  for (int q = 0; q < 4; ++q)
    if (s->cell[q]) m |= 1 << q;
  return m;
}

int popcount4(int m) { return (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1) + ((m >> 3) & 1); }

int upload_axis(yb_sim* s) {
  for (int side = 0; side < 2; ++side) {
    const bool uni = side == 0 ? s->cb_uniform : s->db_uniform;
    const float uv = side == 0 ? s->cb_u : s->db_u;
    for (int a = 0; a < 3; ++a) {
      std::vector<float> h(s->axis_len[a], 0.0f);
      // x, y: full arrays; z: the global array's values for local planes
      // -kGhost..nz+1 (element q + kGhost holds local plane q; ghost planes
      // outside the global grid stay 0 and are never read)
      if (a < 2) {
        for (size_t q = 0; q < s->axis_ref[a].size(); ++q) h[q] = uni ? uv : s->axis_ref[a][q];
      } else {
        const int nzg = (int)s->axis_ref[2].size();
        for (int q = -yb::kGhost; q <= s->g.nz + 1; ++q) {
          const int kg = s->g.zoff + q;
          if (kg >= 0 && kg < nzg) h[q + yb::kGhost] = uni ? uv : s->axis_ref[2][kg];
        }
      }
      YB_CU(cudaMemcpyAsync(s->axis_dev[side * 3 + a], h.data(), h.size() * sizeof(float),
                            cudaMemcpyHostToDevice, s->stream));
    }
  }
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

yb::CoefArgs coef_args(const yb_sim* s) {
  yb::CoefArgs c{};
  for (int q = 0; q < 4; ++q) c.cell[q] = s->cell[q];
  c.ca_s = s->ca_s;
  c.da_s = s->da_s;
  c.cdx_e = s->axis_dev[0];
  c.cdy_e = s->axis_dev[1];
  c.cdz_e = s->axis_dev[2] + yb::kGhost;  // indexable at local planes -kGhost..nz+1
  c.cdx_h = s->axis_dev[3];
  c.cdy_h = s->axis_dev[4];
  c.cdz_h = s->axis_dev[5] + yb::kGhost;
  return c;
}

yb::Fields fields_of(const yb_sim* s, int b) {
  yb::Fields F;
  for (int c = 0; c < 6; ++c) F.f[c] = s->buf[b][c];
  return F;
}

// L2 promotion per kernel, measured (Gcell/s, 3 runs each): the one-step kernel's maps gain with
// 64 B (config 2 96.4 -> 98.6, config 3 87.3 -> 90.6 vs 256 B); the two-step kernel's were best
// or equal with 256 B in row-major item order (config 4 187.1 vs 184.7 with 64 B); see prepare_fused
// for wide grids in column-block order.
constexpr CUtensorMapL2promotion kPromoFused = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
int encode_map(CUtensorMap* m, const Geo& g, float* base, int box_rows = yb::kBY, int box_cols = yb::kBX,
               CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(YB_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  // z coordinate = local plane + kGhost: the allocation starts at ghost plane -kGhost
  const cuuint64_t dims[3] = {(cuuint64_t)g.PX, (cuuint64_t)g.PY, (cuuint64_t)g.PZ + yb::kGhost + 1};
  const cuuint64_t strides[2] = {(cuuint64_t)g.PX * 4, (cuuint64_t)g.plane * 4};
  const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  // YB_L2PROMO=0..3 (tuning knob): none / 64B / 128B / 256B L2 promotion
  if (const char* e = std::getenv("YB_L2PROMO")) promo = (CUtensorMapL2promotion)std::atoi(e);
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base - yb::kGhost * g.plane, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(YB_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return YB_OK;
}

// (Re)build TMA descriptors and the launch shape for the current coefficient set.
int prepare_fused(yb_sim* s) {
  if (s->tm_valid) return YB_OK;
  const int mask = cell_mask(s);
  const int narr = 6 + popcount4(mask);
  for (int b = 0; b < 2; ++b) {
    int q = 0;
    for (int c = 0; c < 6; ++c)
      if (int rc = encode_map(&s->tm[b].m[q++], s->g, s->buf[b][c], yb::kBY, yb::kBX, kPromoFused)) return rc;
    for (int a = 0; a < 4; ++a)
      if (s->cell[a])
        if (int rc = encode_map(&s->tm[b].m[q++], s->g, s->cell[a], yb::kBY, yb::kBX, kPromoFused)) return rc;
  }
  const size_t avail = 227 * 1024;
  // Ring depth: measured best at 4 stages (<= 7 arrays) / 3 (more), i.e.
  // ~150-165 KB in flight per SM; deeper rings lost DRAM efficiency.
  int S = narr <= 7 ? 4 : 3;
  if (const char* e = std::getenv("YB_STAGES")) S = std::max(2, std::min(6, std::atoi(e)));
  while (S > 2 && yb::fused_smem_bytes(narr, S) > avail) --S;
  s->stages = S;
  const int tx = (s->g.nx + yb::kTX - 1) / yb::kTX;
  const int ty = (s->g.ny + yb::kTY - 1) / yb::kTY;
  int zc = s->zchunk_req;
  if (zc <= 0) {
    // Persistent CTAs (one per SM) stride over T*Z items. Minimise the
    // busiest CTA's planes: ceil(T*Z/G) items of (len + ~1.2) planes, the
    // extra being the prologue/epilogue planes a chunk boundary re-reads.
    const long long T = (long long)tx * ty;
    double best = 1e300;
    for (int Z = 1; Z <= s->g.nz; ++Z) {
      const int len = (s->g.nz + Z - 1) / Z;
      const int Zr = (s->g.nz + len - 1) / len;
      const long long rounds = (T * Zr + s->num_sms - 1) / s->num_sms;
      // (1 + len/400): shorter items keep concurrently running neighbours
      // closer in z (halo rows hit L2) and balance better; measured.
      const double cost = (double)rounds * (len + (Zr > 1 ? 1.2 : 0.0)) * (1.0 + len / 400.0);
      if (cost < best - 1e-9) {
        best = cost;
        zc = len;
      }
    }
  }
  zc = std::min(std::max(zc, 1), s->g.nz);
  s->zchunk = zc;
  s->ntx = tx;
  s->nty = ty;
  s->nitems = tx * ty * ((s->g.nz + zc - 1) / zc);
  // YB_CTAS_PER_ITEM=1 (debug/A-B): one CTA per work item instead of persistent CTAs
  const char* one = std::getenv("YB_CTAS_PER_ITEM");
  const int ctas = (one && one[0] == '1') ? s->nitems : std::min(s->nitems, s->num_sms);
  s->grid = dim3(ctas, 1, 1);
  if (s->variant == YB_VARIANT_TB4) {
    for (int b = 0; b < 2; ++b) {
      int q = 0;
      for (int c = 0; c < 6; ++c)
        if (int rc = encode_map(&s->tm4[b].m[q++], s->g, s->buf[b][c], yb::kTB4BY, yb::kTB4Win)) return rc;
      for (int a = 0; a < 4; ++a)
        if (s->cell[a])
          if (int rc = encode_map(&s->tm4[b].m[q++], s->g, s->cell[a], yb::kTB4BY - 1, yb::kTB4Win)) return rc;
    }
    int S4 = 3;
    while (S4 > 2 && yb::tb4_smem_bytes(mask, S4) > avail) --S4;
    s->stages4 = S4;
    s->ntx4 = (s->g.nx + yb::kTB4Cols - 1) / yb::kTB4Cols;
    s->nty4 = (s->g.ny + yb::kTB4Rows - 1) / yb::kTB4Rows;
    int zc4 = s->zchunk_req;
    if (zc4 <= 0) {  // a four-step item re-streams ~7 planes at its z boundaries
      const long long T = (long long)s->ntx4 * s->nty4;
      double best = 1e300;
      for (int Z = 1; Z <= s->g.nz; ++Z) {
        const int len = (s->g.nz + Z - 1) / Z;
        const int Zr = (s->g.nz + len - 1) / len;
        const long long rounds = (T * Zr + s->num_sms - 1) / s->num_sms;
        const double cost = (double)rounds * (len + (Zr > 1 ? 7.0 : 0.0));
        if (cost < best - 1e-9) {
          best = cost;
          zc4 = len;
        }
      }
    }
    s->zchunk4 = std::min(std::max(zc4, 1), s->g.nz);
  }
  if (s->variant == YB_VARIANT_TB2 || s->variant == YB_VARIANT_TB4) {
    // Wide grids (more than 4 tile columns: the sweep's tiles go out in column blocks, so a
    // block's outer x-halo columns miss L2) fetch those columns with 64 B promotion instead of
    // 256 B: config 4 198.8 -> 199.9, config 5 156.5 -> 158.0; up to 4 columns 256 B stays
    // (config 3 162.1 vs 161.2).
    const CUtensorMapL2promotion promo2 =
        tx > 4 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    for (int b = 0; b < 2; ++b) {
      int q = 0;
      for (int c = 0; c < 6; ++c)
        if (int rc = encode_map(&s->tm2[b].m[q++], s->g, s->buf[b][c], yb::tb2_short(c) ? yb::kTB2RowsE : yb::kTB2BY,
                                yb::kBX, promo2))
          return rc;
      for (int a = 0; a < 4; ++a)
        if (s->cell[a])
          if (int rc = encode_map(&s->tm2[b].m[q++], s->g, s->cell[a], a < 2 ? yb::kTB2RowsCA : yb::kTB2RowsDA,
                                  yb::kBX, promo2))
            return rc;
    }
    int S2 = 3;
    if (const char* e = std::getenv("YB_STAGES2")) S2 = std::max(2, std::min(4, std::atoi(e)));
    while (S2 > 2 && yb::tb2_smem_bytes(mask, S2) > avail) --S2;
    s->stages2 = S2;
    int zc2 = s->zchunk_req;
    if (zc2 <= 0) {  // a two-step item re-streams ~3 planes at its z boundaries
      const long long T = (long long)tx * ty;
      double best = 1e300;
      for (int Z = 1; Z <= s->g.nz; ++Z) {
        const int len = (s->g.nz + Z - 1) / Z;
        const int Zr = (s->g.nz + len - 1) / len;
        const long long rounds = (T * Zr + s->num_sms - 1) / s->num_sms;
        const double cost = (double)rounds * (len + (Zr > 1 ? 3.0 : 0.0)) * (1.0 + len / 4000.0);
        if (cost < best - 1e-9) {
          best = cost;
          zc2 = len;
        }
      }
    }
    zc2 = std::min(std::max(zc2, 1), s->g.nz);
    s->zchunk2 = zc2;
    // Multi-sweep launches have no wave tail (the next sweep fills idle SMs),
    // so they take the longest chunks that still leave ~1.7 items per SM in
    // a sweep; each chunk boundary re-streams ~3 planes, so never shorter than
    // 8 planes. Measured (tools/chunk_sweep.sh, Gcell/s): config 1 (128^3,
    // 16 tiles) chunk 4/6/8/10 -> 91/108/114/105 vs 88 with one launch per
    // sweep; config 2 chunk 16/32/52/64 -> 144/163/170/171; configs 3 / 4
    // chunk 64/128/256 -> 157/162/165 and 179/185/187.
    {
      // (~1.7 items per SM and sweep measured best: config 1 chunk 8 -> 256 items, config 2 chunk 64)
      const long long T = (long long)tx * ty, need = (17LL * s->num_sms + 9) / 10;
      // (chunks capped at 256 planes: longer ones measured no better)
      const int Zr = (int)std::min<long long>(s->g.nz, std::max<long long>((need + T - 1) / T, (s->g.nz + 255) / 256));
      const int len = (s->g.nz + Zr - 1) / Zr;
      s->zchunk2p = s->zchunk_req > 0 ? std::min(s->zchunk_req, s->g.nz) : std::max(len, std::min(8, s->g.nz));
    }
    s->nitems2 = tx * ty * ((s->g.nz + zc2 - 1) / zc2);
    s->grid2 = dim3(std::min(s->nitems2, s->num_sms), 1, 1);
  }
  s->tm_valid = true;
  return YB_OK;
}

// Active sources at `step` (and `step+1` when two steps run in one launch).
yb::SrcArgs sources_at(const yb_sim* s, int64_t step, bool two = false) {
  yb::SrcArgs a{};
  for (const Src& q : s->sources) {
    const int64_t n = (int64_t)q.table.size();
    const bool a0 = step >= 0 && step < n, a1 = two && step + 1 >= 0 && step + 1 < n;
    if (!a0 && !a1) continue;
    a.comp[a.n] = q.comp;
    a.i[a.n] = q.i;
    a.j[a.n] = q.j;
    a.k[a.n] = q.k - s->g.zoff;  // local plane (may be outside the slab)
    a.val[a.n] = a0 ? q.table[step] : 0.0f;
    a.val2[a.n] = a1 ? q.table[step + 1] : 0.0f;
    a.act[a.n] = (a0 ? 1 : 0) | (a1 ? 2 : 0);
    ++a.n;
  }
  return a;
}

// Quiescent map for the sweep kernels (nullptr bits when skipping is off).
yb::QMap qmap_of(const yb_sim* s) {
  yb::QMap q{};
  q.ntx = s->ntx;
  q.nty = s->nty;
  q.words = s->qwords;
  q.bits = s->qskip ? s->qbits : nullptr;
  return q;
}

// (Re)builds the quiescent map from both state buffers when it is stale.
int qmap_refresh(yb_sim* s) {
  if (!s->qskip || s->q_valid) return YB_OK;
  const int planes = s->g.nz + 2 * yb::kGhost;  // local planes -kGhost .. nz+kGhost-1
  const int words = (planes + 31) / 32, tiles = s->ntx * s->nty;
  if (words != s->qwords || tiles != s->qtiles) {
    cudaFree(s->qbits);
    s->qbits = nullptr;
    YB_CU(cudaMalloc(&s->qbits, (size_t)tiles * words * 4));
    s->qwords = words;
    s->qtiles = tiles;
  }
  if (!s->qskipped) {
    YB_CU(cudaMalloc(&s->qskipped, sizeof(unsigned long long)));
    YB_CU(cudaMemsetAsync(s->qskipped, 0, sizeof(unsigned long long), s->stream));
  }
  YB_CU(cudaMemsetAsync(s->qbits, 0, (size_t)tiles * words * 4, s->stream));
  YB_CU(yb::launch_qscan(s->g, fields_of(s, 0), fields_of(s, 1), qmap_of(s), -yb::kGhost,
                         s->g.nz + yb::kGhost - 1, s->stream));
  s->q_valid = true;
  return YB_OK;
}

int collect_timers(yb_sim* s) {
  if (s->timers_used == 0) return YB_OK;
  YB_CU(cudaStreamSynchronize(s->stream));
  for (size_t q = 0; q < s->timers_used; ++q) {
    float ms = 0.f;
    YB_CU(cudaEventElapsedTime(&ms, s->timers[q].a, s->timers[q].b));
    s->kernel_ms += ms;
    ++s->kernel_timed;
  }
  s->timers_used = 0;
  return YB_OK;
}

// z-chunk ranges of one sweep launch: [zb0, ze0) then [zb1, ze1).
struct ZPart {
  int zb0, ze0, zb1, ze1;
};
ZPart zfull(const yb_sim* s) { return {0, s->g.nz, s->g.nz, s->g.nz}; }

// Fills the chunk fields of `a`; returns the launch's grid.
dim3 set_chunks(const yb_sim* s, yb::FusedArgs& a, int zchunk, const ZPart& z) {
  const int n0 = z.ze0 > z.zb0 ? (z.ze0 - z.zb0 + zchunk - 1) / zchunk : 0;
  const int n1 = z.ze1 > z.zb1 ? (z.ze1 - z.zb1 + zchunk - 1) / zchunk : 0;
  a.zchunk = zchunk;
  a.zb0 = z.zb0;
  a.ze0 = z.ze0;
  a.zb1 = z.zb1;
  a.ze1 = z.ze1;
  a.nch0 = n0;
  a.nitems = s->ntx * s->nty * (n0 + n1);
  const char* one = std::getenv("YB_CTAS_PER_ITEM");
  return dim3((one && one[0] == '1') ? a.nitems : std::min(a.nitems, s->num_sms), 1, 1);
}

int step_fused(yb_sim* s, ZPart z, int zchunk, bool flip) {
  const int nxt = s->cur ^ 1;
  yb::FusedArgs a{};
  a.g = s->g;
  a.nstages = s->stages;
  a.ntx = s->ntx;
  a.nty = s->nty;
  const dim3 grid = set_chunks(s, a, zchunk, z);
  cudaStream_t st = s->on_side ? s->side : s->stream;
  unsigned long long* sc = s->on_side ? s->sched2 : s->sched;
  unsigned long long& base = s->on_side ? s->sched2_base : s->sched_base;
  a.sched = sc;
  a.sched_base = base;
  a.no_faces = s->on_side ? 1 : 0;  // the boundary launch of the split sweep does them
  a.store_policy = s->store_policy;
  a.co = coef_args(s);
  for (int c = 0; c < 6; ++c) {
    a.in[c] = s->buf[s->cur][c];
    a.out[c] = s->buf[nxt][c];
  }
  a.src = sources_at(s, s->step_index);
  a.qm = qmap_of(s);
  a.skipped = s->qskipped;
  const int mask = cell_mask(s);
  const size_t smem = yb::fused_smem_bytes(6 + popcount4(mask), s->stages);
  TimerPair* tp = nullptr;
  if (s->timing) {
    if (s->timers_used == s->timers.size()) {
      TimerPair p;
      YB_CU(cudaEventCreate(&p.a));
      YB_CU(cudaEventCreate(&p.b));
      s->timers.push_back(p);
    }
    tp = &s->timers[s->timers_used++];
    YB_CU(cudaEventRecord(tp->a, st));
  }
  YB_CU(yb::launch_fused(a, s->tm[s->cur], mask, grid, smem, st));
  base += (unsigned long long)a.nitems + grid.x;  // every CTA's last fetch fails
  if (tp) YB_CU(cudaEventRecord(tp->b, st));
  s->launches += 1;
  if (flip) s->cur = nxt;
  if (s->timers_used >= 4096) return collect_timers(s);
  return YB_OK;
}

// Two Standard steps in one launch (temporal depth 2).
int step_tb2(yb_sim* s, ZPart z, int zchunk, bool flip, int nsweeps = 1) {
  const int nxt = s->cur ^ 1;
  yb::FusedArgs a{};
  a.g = s->g;
  a.nstages = s->stages2;
  a.pf = s->pf2;
  a.ntx = s->ntx;
  a.nty = s->nty;
  const dim3 grid = set_chunks(s, a, zchunk, z);
  cudaStream_t st = s->on_side ? s->side : s->stream;
  unsigned long long* sc = s->on_side ? s->sched2 : s->sched;
  unsigned long long& base = s->on_side ? s->sched2_base : s->sched_base;
  a.nsweeps = nsweeps;
  a.err = s->werr;
  a.wait_ns = s->wait_ns;
  if (s->peer_stores) {  // MODE 3: boundary planes straight into the neighbours' (same-parity) buffers
    for (int c = 0; c < 6; ++c) {
      a.pdn[c] = s->peer[0].on ? s->peer[0].buf[nxt][c] : nullptr;
      a.pup[c] = s->peer[1].on ? s->peer[1].buf[nxt][c] : nullptr;
    }
    a.pdn_k0 = s->peer[0].nz;
    // Fold the wait / signal into the launch when only the bottom / top z-chunk
    // touches the ghost planes (both at least two planes deep); else separate
    // wait and signal launches around it.
    const int T = a.ntx * a.nty, nch = a.nitems / T;
    auto planes = [&](int c, int& k0, int& k1) {
      if (c < a.nch0) {
        k0 = a.zb0 + c * a.zchunk;
        k1 = std::min(k0 + a.zchunk, a.ze0);
      } else {
        k0 = a.zb1 + (c - a.nch0) * a.zchunk;
        k1 = std::min(k0 + a.zchunk, a.ze1);
      }
    };
    int f0, f1, l0, l1;
    planes(0, f0, f1);
    planes(nch - 1, l0, l1);
    s->peer_folded = !s->on_side && f0 == 0 && f1 - f0 >= 2 && l1 == s->g.nz && l1 - l0 >= 2 &&
                     std::getenv("YB_PEER_NOFOLD") == nullptr;
    if (s->peer_folded) {
      if (s->peer_inflight) {  // my own push must have read my planes before they are rewritten
        YB_CU(cudaStreamWaitEvent(st, s->peer_done, 0));
        s->peer_inflight = false;
      }
      a.pfold = std::getenv("YB_PEER_NOREMAP") ? 2 : 1;
      a.pflag = s->pflags;
      a.pneed = s->push_count;
      a.psig_val = s->push_count + 1;
      a.psig[0] = s->peer[0].on ? s->peer[0].flags + 1 : nullptr;
      a.psig[1] = s->peer[1].on ? s->peer[1].flags + 0 : nullptr;
      a.pcnt = s->pflags + 4;
      a.pcnt_base[0] = s->pcnt_base[0];
      a.pcnt_base[1] = s->pcnt_base[1];
      a.perr = s->werr;
      if (s->peer[0].on) s->pcnt_base[0] += (unsigned)T * yb::kTB2RowWarps;  // every row warp counts
      if (s->peer[1].on) s->pcnt_base[1] += (unsigned)T * yb::kTB2RowWarps;
    } else {
      if (int rc = yb_peer_wait(s)) return rc;
    }
  }
  if (nsweeps > 1) {  // several sweeps in one launch, items ordered by dependency
    if (s->done_n != a.nitems) {
      cudaFree(s->done);
      s->done = nullptr;
      YB_CU(cudaMalloc(&s->done, (size_t)a.nitems * sizeof(unsigned)));
      YB_CU(cudaMemsetAsync(s->done, 0, (size_t)a.nitems * sizeof(unsigned), s->stream));
      s->done_n = a.nitems;
      s->epoch = 0;
    }
    if (s->srcs_cap < nsweeps) {
      cudaFree(s->srcs_dev);
      s->srcs_dev = nullptr;
      YB_CU(cudaMalloc(&s->srcs_dev, (size_t)nsweeps * sizeof(yb::SrcArgs)));
      s->srcs_cap = nsweeps;
    }
    std::vector<yb::SrcArgs> sv(nsweeps);
    for (int q = 0; q < nsweeps; ++q) sv[q] = sources_at(s, s->step_index + 2 * q, true);
    YB_CU(cudaMemcpyAsync(s->srcs_dev, sv.data(), sv.size() * sizeof(yb::SrcArgs), cudaMemcpyHostToDevice,
                          s->stream));
    a.done = s->done;
    a.epoch = s->epoch;
    a.srcs = s->srcs_dev;
    a.xblock = s->xblock;
    if (s->drain) {  // streamed readback: skewed last sweeps, band counters (set up by yb_run_to_host)
      a.diag = s->diag_dev;
      a.ndiag = s->ndiag;
      a.skew0 = nsweeps - s->diag_sweeps;
      a.band = s->band_dev;
    }
    if (s->upstream) {  // streamed upload: skewed first sweeps behind the copies (yb_run_streamed)
      a.skewh = s->diagh_sweeps;
      a.diagh = s->diagh_dev;
      a.ndiagh = s->ndiagh;
      a.upband = s->upband_dev;
      a.up_need = s->up_base + 1;
    }
  }
  a.sched = sc;
  a.sched_base = base;
  a.no_faces = s->on_side ? 1 : 0;  // the boundary launch of the split sweep does them
  a.store_policy = 1;
  a.co = coef_args(s);
  for (int c = 0; c < 6; ++c) {
    a.in[c] = s->buf[s->cur][c];
    a.out[c] = s->buf[nxt][c];
  }
  a.src = sources_at(s, s->step_index, true);
  a.qm = qmap_of(s);
  a.skipped = s->qskipped;
  const int mask = cell_mask(s);
  const size_t smem = yb::tb2_smem_bytes(mask, s->stages2);
  TimerPair* tp = nullptr;
  if (s->timing) {
    if (s->timers_used == s->timers.size()) {
      TimerPair p;
      YB_CU(cudaEventCreate(&p.a));
      YB_CU(cudaEventCreate(&p.b));
      s->timers.push_back(p);
    }
    tp = &s->timers[s->timers_used++];
    YB_CU(cudaEventRecord(tp->a, st));
  }
#ifdef YB_TB2_STAMP
  unsigned long long* stamp_dev = nullptr;
  const char* stamp_file = std::getenv("YB_TB2_STAMP_FILE");
  const size_t stamp_n = 2 * (size_t)a.nitems * nsweeps;
  if (stamp_file && nsweeps > 1) {
    YB_CU(cudaMalloc(&stamp_dev, stamp_n * 8));
    YB_CU(cudaMemsetAsync(stamp_dev, 0, stamp_n * 8, st));
    a.stamp = stamp_dev;
  }
#endif
  YB_CU(yb::launch_tb2(a, s->tm2[s->cur], s->tm2[nxt], mask, grid, smem, st));
#ifdef YB_TB2_STAMP
  if (stamp_dev) {
    std::vector<unsigned long long> h(stamp_n);
    YB_CU(cudaStreamSynchronize(st));
    YB_CU(cudaMemcpy(h.data(), stamp_dev, stamp_n * 8, cudaMemcpyDeviceToHost));
    cudaFree(stamp_dev);
    if (FILE* f = std::fopen(stamp_file, "wb")) {
      const int hdr[6] = {a.nitems, nsweeps, a.ntx, a.nty, a.zchunk, s->g.nz};
      std::fwrite(hdr, sizeof hdr, 1, f);
      std::fwrite(h.data(), 8, stamp_n, f);
      std::fclose(f);
    }
  }
#endif
  s->last_grid = grid.x;
  base += (unsigned long long)a.nitems * nsweeps + grid.x;
  if (nsweeps > 1) s->epoch += (unsigned)nsweeps;
  if (tp) YB_CU(cudaEventRecord(tp->b, st));
  s->launches += 1;
  if (flip && (nsweeps & 1)) s->cur = nxt;
  if (s->timers_used >= 4096) return collect_timers(s);
  return YB_OK;
}

// Active sources of steps step .. step+3 (the four steps of one depth-4 launch).
yb::SrcArgs4 sources_at4(const yb_sim* s, int64_t step) {
  yb::SrcArgs4 a{};
  for (const Src& q : s->sources) {
    const int64_t n = (int64_t)q.table.size();
    int act = 0;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < 4; ++t)
      if (step + t >= 0 && step + t < n) {
        act |= 1 << t;
        v[t] = q.table[step + t];
      }
    if (!act) continue;
    a.comp[a.n] = q.comp;
    a.i[a.n] = q.i;
    a.j[a.n] = q.j;
    a.k[a.n] = q.k - s->g.zoff;
    for (int t = 0; t < 4; ++t) a.val[a.n][t] = v[t];
    a.act[a.n] = act;
    ++a.n;
  }
  return a;
}

// Four Standard steps in one launch (temporal depth 4, single domain).
int step_tb4(yb_sim* s) {
  const int nxt = s->cur ^ 1;
  yb::FusedArgs a{};
  a.g = s->g;
  a.nstages = s->stages4;
  a.ntx = s->ntx4;
  a.nty = s->nty4;
  a.zchunk = s->zchunk4;
  a.zb0 = 0, a.ze0 = s->g.nz, a.zb1 = a.ze1 = s->g.nz;
  a.nch0 = (s->g.nz + s->zchunk4 - 1) / s->zchunk4;
  a.nitems = s->ntx4 * s->nty4 * a.nch0;
  a.sched = s->sched;
  a.sched_base = s->sched_base;
  a.co = coef_args(s);
  for (int c = 0; c < 6; ++c) {
    a.in[c] = s->buf[s->cur][c];
    a.out[c] = s->buf[nxt][c];
  }
  const yb::SrcArgs4 src = sources_at4(s, s->step_index);
  const int mask = cell_mask(s);
  const dim3 grid(std::min(a.nitems, s->num_sms), 1, 1);
  TimerPair* tp = nullptr;
  if (s->timing) {
    if (s->timers_used == s->timers.size()) {
      TimerPair p;
      YB_CU(cudaEventCreate(&p.a));
      YB_CU(cudaEventCreate(&p.b));
      s->timers.push_back(p);
    }
    tp = &s->timers[s->timers_used++];
    YB_CU(cudaEventRecord(tp->a, s->stream));
  }
  YB_CU(yb::launch_tb4(a, src, s->tm4[s->cur], mask, grid, yb::tb4_smem_bytes(mask, s->stages4), s->stream));
  s->sched_base += (unsigned long long)a.nitems + grid.x;
  if (tp) YB_CU(cudaEventRecord(tp->b, s->stream));
  s->launches += 1;
  s->cur = nxt;
  s->q_valid = false;  // this kernel does not maintain the quiescent map
  if (s->timers_used >= 4096) return collect_timers(s);
  return YB_OK;
}

int step_naive(yb_sim* s) {
  const int box[6] = {0, s->g.nx + 1, 0, s->g.ny + 1, 0, s->g.nz + 1};
  const yb::Fields F = fields_of(s, s->cur);
  const yb::CoefArgs co = coef_args(s);
  TimerPair* tp = nullptr;
  if (s->timing) {
    if (s->timers_used == s->timers.size()) {
      TimerPair p;
      YB_CU(cudaEventCreate(&p.a));
      YB_CU(cudaEventCreate(&p.b));
      s->timers.push_back(p);
    }
    tp = &s->timers[s->timers_used++];
    YB_CU(cudaEventRecord(tp->a, s->stream));
  }
  YB_CU(yb::launch_naive_ampere(s->g, F, co, box, s->stream));
  YB_CU(yb::launch_naive_pec(s->g, F, s->stream));
  const yb::SrcArgs src = sources_at(s, s->step_index);
  int n = 3;
  if (src.n) {
    YB_CU(yb::launch_sources(s->g, F, src, s->stream));
    ++n;
  }
  YB_CU(yb::launch_naive_faraday(s->g, F, co, box, s->stream));
  if (tp) YB_CU(cudaEventRecord(tp->b, s->stream));
  s->launches += n;
  if (s->timers_used >= 4096) return collect_timers(s);
  return YB_OK;
}

int check_comp(int comp) {
  if (comp < 0 || comp > 5) return fail(YB_INVALID_ARGUMENT, "component %d out of [0,5]", comp);
  return YB_OK;
}

// Host <-> device transfer of one dense reference-layout array through a
// staging buffer: one linear cudaMemcpy at full link speed plus a device
// scatter/gather into the padded node box (pitched 3D copies of short rows
// run far below link speed). The staging buffer is the next-state buffer of
// the same component, re-zeroed afterwards (its DoFs are rewritten by the
// next step; its non-DoF positions must stay +0).
int copy_dense(yb_sim* s, int comp, float* dev, const float* hsrc, float* hdst) {
  int e[3];
  comp_ext(s->g, comp, e);
  const size_t n = (size_t)e[0] * e[1] * e[2];
  float* stage = s->buf[s->cur ^ 1][comp];
  if (hsrc) {
    YB_CU(yb::copy_h2d(stage, hsrc, n * 4, s->stream));
    YB_CU(yb::launch_scatter_dense(s->g, e, stage, dev, s->stream));
  } else {
    YB_CU(yb::launch_gather_dense(s->g, e, dev, stage, s->stream));
    YB_CU(yb::copy_d2h(hdst, stage, n * 4, s->stream));
  }
  YB_CU(cudaMemsetAsync(stage - yb::kGhost * s->g.plane, 0, (size_t)s->g.total * 4, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

float courant() {
  const uint32_t b = YB_S_BITS;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

}  // namespace

extern "C" {

const char* yb_last_error(void) { return g_err.c_str(); }
int yb_abi_version(void) { return YB_ABI_VERSION; }

int yb_create(const yb_desc* d, yb_sim** out) {
  if (!d || !out) return fail(YB_INVALID_ARGUMENT, "yb_create: null argument");
  *out = nullptr;
  if (d->nx < 1 || d->ny < 1 || d->nz < 1)
    return fail(YB_INVALID_ARGUMENT, "GridSpec: cell counts must be positive");
  if (d->ny > 65000 || d->nz > 65000 || d->nx > (1 << 24))
    return fail(YB_INVALID_ARGUMENT, "grid too large for this build");
  if (d->variant != YB_VARIANT_FUSED && d->variant != YB_VARIANT_NAIVE &&
      d->variant != YB_VARIANT_TB2 && d->variant != YB_VARIANT_TB4)
    return fail(YB_INVALID_ARGUMENT, "unknown variant %d", d->variant);
  if (d->variant == YB_VARIANT_TB4 && d->nz_global > 0 && d->nz_global != d->nz)
    return fail(YB_INVALID_ARGUMENT, "the four-step variant works on a single domain (no z-slabs)");
  if (d->nz_global > 0 && (d->z_offset < 0 || d->z_offset + d->nz > d->nz_global))
    return fail(YB_INVALID_ARGUMENT, "slab [%d,%d) outside the global grid of %d planes",
                d->z_offset, d->z_offset + d->nz, d->nz_global);
  if (d->nz_global <= 0 && d->z_offset != 0)
    return fail(YB_INVALID_ARGUMENT, "z_offset needs nz_global");
  if (d->nz_global > 0 && d->nz_global != d->nz && d->variant == YB_VARIANT_NAIVE)
    return fail(YB_INVALID_ARGUMENT, "z-slab mode needs a sweep variant (FUSED or TB2)");
  if (d->nz_global > 0 && d->nz_global != d->nz && d->nz < 2)
    return fail(YB_INVALID_ARGUMENT, "z-slabs need at least 2 planes each");
  YB_CU(cudaSetDevice(d->device));
  yb_sim* s = new yb_sim;
  s->device = d->device;
  s->variant = d->variant;
  s->zchunk_req = d->zchunk;
  if (const char* e = std::getenv("YB_STPOL")) s->store_policy = std::atoi(e);
  if (const char* e = std::getenv("YB_TB2_PERSIST")) s->persist = std::atoi(e) != 0;
  if (const char* e = std::getenv("YB_TB2_PF")) s->pf2 = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("YB_TB2_XBLOCK")) s->xblock = std::max(0, std::atoi(e));
  Geo& g = s->g;
  g.nx = d->nx;
  g.ny = d->ny;
  g.nz = d->nz;
  g.zoff = d->z_offset;
  g.nzg = d->nz_global > 0 ? d->nz_global : d->nz;
  g.PX = ((d->nx + 1 + 31) / 32) * 32;
  g.PY = d->ny + 1;
  g.PZ = d->nz + 1;
  g.plane = (long long)g.PX * g.PY;
  g.total = g.plane * (g.PZ + yb::kGhost + 2);  // planes -2..nz+1 + 1 guard plane
  int dev_sms = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, d->device);
  if (dev_sms > 0) s->num_sms = dev_sms;
  auto bail = [&](int rc) {
    yb_destroy(s);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(YB_CUDA_ERROR, "stream create failed"));
  s->stream = s->own_stream;
  // the transfer side stream exists from the start (not created inside a timed upload)
  if (cudaStreamCreateWithFlags(&s->xfer, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(YB_CUDA_ERROR, "stream create failed"));
  for (cudaEvent_t& e : s->xev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(YB_CUDA_ERROR, "event create failed"));
  const size_t bytes = (size_t)g.total * sizeof(float);
  for (int b = 0; b < 2; ++b)
    for (int c = 0; c < 6; ++c) {
      float* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess)
        return bail(fail(YB_CUDA_ERROR, "cudaMalloc of %zu bytes failed", bytes));
      s->buf[b][c] = p + yb::kGhost * g.plane;
      s->dev_bytes += bytes;
      if (cudaMemsetAsync(p, 0, bytes, s->stream) != cudaSuccess)
        return bail(fail(YB_CUDA_ERROR, "memset failed"));
    }
  const int ns[3] = {g.nx, g.ny, g.nz};
  for (int a = 0; a < 3; ++a) {
    s->axis_len[a] = ((ns[a] + yb::kTX) / yb::kTX + 1) * yb::kTX + 64 + yb::kGhost;
    s->axis_ref[a].assign(a == 2 ? g.nzg : ns[a], 0.0f);  // z: the global array
  }
  for (int q = 0; q < 6; ++q) {
    const size_t ab = (size_t)s->axis_len[q % 3] * sizeof(float);
    if (cudaMalloc(&s->axis_dev[q], ab) != cudaSuccess)
      return bail(fail(YB_CUDA_ERROR, "cudaMalloc failed"));
    s->dev_bytes += ab;
  }
  if (cudaMalloc(&s->sched, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemsetAsync(s->sched, 0, 4 * sizeof(unsigned long long), s->stream) != cudaSuccess)
    return bail(fail(YB_CUDA_ERROR, "scheduler counter alloc failed"));
  if (cudaMalloc(&s->werr, 8 * sizeof(int)) != cudaSuccess ||
      cudaMemsetAsync(s->werr, 0, 8 * sizeof(int), s->stream) != cudaSuccess)
    return bail(fail(YB_CUDA_ERROR, "wait-error record alloc failed"));
  if (const char* w = std::getenv("YB_WAIT_TIMEOUT_MS")) {
    const long long ms = std::atoll(w);
    if (ms > 0) s->wait_ns = (unsigned long long)ms * 1000000ull;
  }
  if (int rc = upload_axis(s)) return bail(rc);
  static bool limits_set = false;
  if (!limits_set) {
    if (yb::fused_set_smem_limits() != cudaSuccess || yb::tb2_set_smem_limits() != cudaSuccess ||
        yb::tb4_set_smem_limits() != cudaSuccess)
      return bail(fail(YB_CUDA_ERROR, "cudaFuncSetAttribute failed"));
    limits_set = true;
  }
  if (cudaStreamSynchronize(s->stream) != cudaSuccess)
    return bail(fail(YB_CUDA_ERROR, "init sync failed"));
  *out = s;
  return YB_OK;
}

int yb_destroy(yb_sim* s) {
  if (!s) return YB_OK;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int b = 0; b < 2; ++b)
    for (int c = 0; c < 6; ++c)
      if (s->buf[b][c]) cudaFree(s->buf[b][c] - yb::kGhost * s->g.plane);
  for (int q = 0; q < 4; ++q)
    if (s->cell[q]) cudaFree(s->cell[q] - yb::kGhost * s->g.plane);
  for (int q = 0; q < 6; ++q) cudaFree(s->axis_dev[q]);
  cudaFree(s->sched);
  cudaFree(s->sched2);
  if (s->pcnt4) cudaFree(s->pcnt4);
  if (s->chain_ev) cudaEventDestroy(s->chain_ev);
  cudaFree(s->werr);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->xfer) cudaStreamDestroy(s->xfer);
  if (s->cflags) cudaFree(s->cflags);
  for (cudaEvent_t e : s->xev)
    if (e) cudaEventDestroy(e);
  if (s->ev_pre) cudaEventDestroy(s->ev_pre);
  if (s->ev_int) cudaEventDestroy(s->ev_int);
  cudaFree(s->probe_dev);
  cudaFree(s->qbits);
  cudaFree(s->qskipped);
  cudaFree(s->upband_dev);
  cudaFree(s->diagh_dev);
  cudaFree(s->done);
  cudaFree(s->srcs_dev);
  cudaFree(s->diag_dev);
  cudaFree(s->band_dev);
  for (float* p : s->snap_h) cudaFree(p);
  for (PeerSide& ps : s->peer)
    for (void* p : ps.ipc) cudaIpcCloseMemHandle(p);
  cudaFree(s->pflags);
  if (s->peer_stream) cudaStreamDestroy(s->peer_stream);
  if (s->peer_go) cudaEventDestroy(s->peer_go);
  if (s->peer_done) cudaEventDestroy(s->peer_done);
  cudaFree(s->energy_dev);
  for (auto& t : s->timers) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
  return YB_OK;
}

int yb_set_axis_coeffs(yb_sim* s, const float* cdx, const float* cdy, const float* cdz) {
  if (!s || !cdx || !cdy || !cdz) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  s->axis_ref[0].assign(cdx, cdx + s->g.nx);
  s->axis_ref[1].assign(cdy, cdy + s->g.ny);
  s->axis_ref[2].assign(cdz, cdz + s->g.nzg);
  return upload_axis(s);
}

// Per-cell coefficient upload, part 1: the host array into a staging buffer
// and a device check of uniformity (bit patterns) into *flag; no sync.
static int cell_stage(yb_sim* s, const float* cells, long long n, float* stage, int* flag) {
  YB_CU(yb::copy_h2d(stage, cells, (size_t)n * 4, s->stream));
  const int one = 1;
  YB_CU(cudaMemcpyAsync(flag, &one, 4, cudaMemcpyHostToDevice, s->stream));
  YB_CU(yb::launch_all_equal(stage, n, flag, s->num_sms, s->stream));
  return YB_OK;
}

static long long cell_count(const yb_sim* s) {
  // single domain: nz cell planes. z-slab mode: nz + 2*kGhost planes, the
  // global cell planes z_offset-kGhost .. z_offset+nz+kGhost-1 (entries of
  // planes outside the global grid are ignored)
  const int nzc = s->g.nzg != s->g.nz ? s->g.nz + 2 * yb::kGhost : s->g.nz;
  return (long long)s->g.nx * s->g.ny * nzc;
}

// Part 2: store array `which` from the staged copy (or as a uniform value).
static int cell_finish(yb_sim* s, int which, const float* cells, bool all_equal, float v, float* stage) {
  const bool slab = s->g.nzg != s->g.nz;
  const int nzc = slab ? s->g.nz + 2 * yb::kGhost : s->g.nz;
  s->tm_valid = false;
  if ((which == YB_CA || which == YB_DA) && (!cells || all_equal) && v != 1.0f) {
    // a uniform Ca / Da other than 1 is stored as a full array: the sweep
    // kernels treat "no Ca/Da array" as exactly 1 and skip the multiply
    if (cells) YB_CU(cudaMemsetAsync(stage, 0, (size_t)s->g.total * 4, s->stream));
    if (!s->cell[which]) {
      float* p = nullptr;
      YB_CU(cudaMalloc(&p, (size_t)s->g.total * 4));
      s->cell[which] = p + yb::kGhost * s->g.plane;
      s->dev_bytes += (size_t)s->g.total * 4;
    }
    YB_CU(yb::launch_fill_value(s->cell[which] - yb::kGhost * s->g.plane, s->g.total, v, s->stream));
    if (which == YB_CA) s->ca_s = 1.0f;
    if (which == YB_DA) s->da_s = 1.0f;
    YB_CU(cudaStreamSynchronize(s->stream));
    return YB_OK;
  }
  if (!cells || all_equal) {
    if (cells) YB_CU(cudaMemsetAsync(stage, 0, (size_t)s->g.total * 4, s->stream));
    if (s->cell[which]) {
      YB_CU(cudaFree(s->cell[which] - yb::kGhost * s->g.plane));
      s->cell[which] = nullptr;
      s->dev_bytes -= (size_t)s->g.total * 4;
    }
    if (which == YB_CA) s->ca_s = v;
    if (which == YB_DA) s->da_s = v;
    if (which == YB_CB) {
      s->cb_uniform = cells != nullptr;
      s->cb_u = v;
    }
    if (which == YB_DB) {
      s->db_uniform = cells != nullptr;
      s->db_u = v;
    }
    if (which == YB_CB || which == YB_DB) return upload_axis(s);
    return YB_OK;
  }
  if (which == YB_CB) s->cb_uniform = false;
  if (which == YB_DB) s->db_uniform = false;
  if (!s->cell[which]) {
    float* p = nullptr;
    YB_CU(cudaMalloc(&p, (size_t)s->g.total * 4));
    YB_CU(cudaMemsetAsync(p, 0, (size_t)s->g.total * 4, s->stream));
    s->cell[which] = p + yb::kGhost * s->g.plane;
    s->dev_bytes += (size_t)s->g.total * 4;
  }
  const int ce[3] = {s->g.nx, s->g.ny, nzc};
  float* dst = slab ? s->cell[which] - yb::kGhost * s->g.plane : s->cell[which];
  YB_CU(yb::launch_scatter_dense(s->g, ce, stage, dst, s->stream));
  YB_CU(yb::launch_clamp_fill(s->g, s->cell[which], slab ? -yb::kGhost : 0,
                              slab ? s->g.nz + 1 : nzc - 1, s->stream));
  YB_CU(cudaMemsetAsync(stage, 0, (size_t)s->g.total * 4, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_set_cell_coeffs(yb_sim* s, int which, const float* cells, float uniform) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (which < 0 || which > 3) return fail(YB_INVALID_ARGUMENT, "coefficient selector %d", which);
  if (cells) return yb_set_cell_coeffs_n(s, 1, &which, &cells);
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  return cell_finish(s, which, nullptr, false, uniform, nullptr);
}

int yb_set_cell_coeffs_n(yb_sim* s, int n, const int* which, const float* const* cells) {
  if (!s || !which || !cells) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (n < 1 || n > 4) return fail(YB_INVALID_ARGUMENT, "1 .. 4 arrays (got %d)", n);
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  for (int i = 0; i < n; ++i) {
    if (which[i] < 0 || which[i] > 3 || !cells[i]) return fail(YB_INVALID_ARGUMENT, "bad array %d", i);
    for (int k = 0; k < i; ++k)
      if (which[k] == which[i]) return fail(YB_INVALID_ARGUMENT, "coefficient %d given twice", which[i]);
  }
  YB_CU(cudaSetDevice(s->device));
  if (!s->cflags) YB_CU(cudaMalloc(&s->cflags, 4 * sizeof(int)));
  // Staging: the spare state buffers from their allocation start (see
  // copy_dense; re-zeroed after use). With peer links the neighbours may be
  // storing into this handle's spare buffer's ghost planes, so each array
  // goes through a scratch allocation instead.
  const bool scratch = s->peer[0].on || s->peer[1].on;
  float* stage[4] = {};
  auto cleanup = [&](int rc) {
    for (int i = 0; i < n; ++i) {
      if (!stage[i]) continue;
      if (scratch)
        cudaFree(stage[i]);
      else if (rc != YB_OK)  // an error left staged data behind: restore the +0 invariant
        cudaMemsetAsync(stage[i], 0, (size_t)s->g.total * 4, s->stream);
    }
    if (rc != YB_OK || scratch) cudaStreamSynchronize(s->stream);
    return rc;
  };
  // all copies back to back, then one sync for the uniformity checks
  for (int i = 0; i < n; ++i) {
    if (scratch) {
      if (cudaMalloc(&stage[i], (size_t)s->g.total * 4) != cudaSuccess)
        return cleanup(fail(YB_CUDA_ERROR, "coefficient staging buffer: cudaMalloc failed"));
    } else {
      stage[i] = s->buf[s->cur ^ 1][i] - yb::kGhost * s->g.plane;
    }
    if (int rc = cell_stage(s, cells[i], cell_count(s), stage[i], s->cflags + i)) return cleanup(rc);
  }
  int same[4] = {0, 0, 0, 0};
  if (cudaMemcpyAsync(same, s->cflags, n * sizeof(int), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
      cudaStreamSynchronize(s->stream) != cudaSuccess)
    return cleanup(fail(YB_CUDA_ERROR, "coefficient uniformity check failed"));
  for (int i = 0; i < n; ++i)
    if (int rc = cell_finish(s, which[i], cells[i], same[i] != 0, cells[i][0], stage[i])) return cleanup(rc);
  return cleanup(YB_OK);
}

int yb_generate_medium(yb_sim* s, int64_t eps_seed, int64_t sigma_seed) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  const float S = courant();
  s->tm_valid = false;
  auto ensure = [&](int q) -> int {
    if (!s->cell[q]) {
      float* p = nullptr;
      YB_CU(cudaMalloc(&p, (size_t)s->g.total * 4));
      YB_CU(cudaMemsetAsync(p, 0, (size_t)s->g.total * 4, s->stream));
      s->cell[q] = p + yb::kGhost * s->g.plane;
      s->dev_bytes += (size_t)s->g.total * 4;
    }
    return YB_OK;
  };
  auto drop = [&](int q) -> int {
    if (s->cell[q]) {
      YB_CU(cudaFree(s->cell[q] - yb::kGhost * s->g.plane));
      s->cell[q] = nullptr;
      s->dev_bytes -= (size_t)s->g.total * 4;
    }
    return YB_OK;
  };
  if (eps_seed < 0 && sigma_seed < 0) {  // vacuum: the grid's own coefficients
    for (int q = 0; q < 4; ++q)
      if (int rc = drop(q)) return rc;
    s->ca_s = s->da_s = 1.0f;
    s->cb_uniform = s->db_uniform = false;
    return upload_axis(s);
  }
  if (sigma_seed < 0) {  // lossless dielectric: Ca = Da = 1, Db = S exactly
    for (int q : {YB_CA, YB_DA, YB_DB})
      if (int rc = drop(q)) return rc;
    if (int rc = ensure(YB_CB)) return rc;
    s->ca_s = s->da_s = 1.0f;
    s->cb_uniform = false;
    s->db_uniform = true;
    s->db_u = S;
    YB_CU(yb::launch_medium(s->g, nullptr, s->cell[YB_CB], nullptr, nullptr, eps_seed, sigma_seed,
                            S, s->stream));
    return upload_axis(s);
  }
  for (int q = 0; q < 4; ++q)
    if (int rc = ensure(q)) return rc;
  s->cb_uniform = s->db_uniform = false;
  YB_CU(yb::launch_medium(s->g, s->cell[0], s->cell[1], s->cell[2], s->cell[3], eps_seed,
                          sigma_seed, S, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_host_medium(int nx, int ny, int nz, int64_t eps_seed, int64_t sigma_seed, float* ca,
                   float* cb, float* da, float* db) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(YB_INVALID_ARGUMENT, "bad grid");
  const float S = courant();
  const long long n = (long long)nx * ny * nz;
  for (long long q = 0; q < n; ++q) {
    const yb_cell_coeffs c = yb_cell_coeffs_at(eps_seed, sigma_seed, (uint64_t)q, S);
    if (ca) ca[q] = c.ca;
    if (cb) cb[q] = c.cb;
    if (da) da[q] = c.da;
    if (db) db[q] = c.db;
  }
  return YB_OK;
}

int yb_host_field(int nx, int ny, int nz, uint64_t seed, int comp, float* dense) {
  if (nx < 1 || ny < 1 || nz < 1 || !dense) return fail(YB_INVALID_ARGUMENT, "bad argument");
  if (int rc = check_comp(comp)) return rc;
  Geo g{};
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  int e[3];
  comp_ext(g, comp, e);
  const long long n = (long long)e[0] * e[1] * e[2];
  for (long long q = 0; q < n; ++q) dense[q] = yb_field_value(seed, comp, (uint64_t)q);
  return YB_OK;
}

int yb_host_field_slab(int nx, int ny, int nz_global, int z_offset, int nplanes, uint64_t seed,
                       int comp, float* dense) {
  if (nx < 1 || ny < 1 || nz_global < 1 || !dense || z_offset < 0 || nplanes < 0)
    return fail(YB_INVALID_ARGUMENT, "bad argument");
  if (int rc = check_comp(comp)) return rc;
  Geo g{};
  g.nx = nx;
  g.ny = ny;
  g.nz = nz_global;
  int e[3];
  comp_ext(g, comp, e);
  const long long pl = (long long)e[0] * e[1];
  for (int k = 0; k < nplanes; ++k) {
    const int kg = z_offset + k;
    for (long long q = 0; q < pl; ++q)
      dense[k * pl + q] = kg < e[2] ? yb_field_value(seed, comp, (uint64_t)(kg * pl + q)) : 0.0f;
  }
  return YB_OK;
}

int yb_host_medium_slab(int nx, int ny, int nz_global, int z_offset, int nplanes,
                        int64_t eps_seed, int64_t sigma_seed, float* ca, float* cb, float* da,
                        float* db) {
  if (nx < 1 || ny < 1 || nz_global < 1 || nplanes < 0) return fail(YB_INVALID_ARGUMENT, "bad argument");
  const float S = courant();
  const long long pl = (long long)nx * ny;
  for (int k = 0; k < nplanes; ++k) {  // cell planes outside the grid: clamped copies
    const long long kg = std::max(0, std::min(z_offset + k, nz_global - 1));
    for (long long q = 0; q < pl; ++q) {
      const yb_cell_coeffs c = yb_cell_coeffs_at(eps_seed, sigma_seed, (uint64_t)(kg * pl + q), S);
      const long long o = k * pl + q;
      if (ca) ca[o] = c.ca;
      if (cb) cb[o] = c.cb;
      if (da) da[o] = c.da;
      if (db) db[o] = c.db;
    }
  }
  return YB_OK;
}

int yb_upload_field(yb_sim* s, int comp, const float* dense) {
  if (!s || !dense) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (int rc = check_comp(comp)) return rc;
  YB_CU(cudaSetDevice(s->device));
  s->q_valid = false;
  return copy_dense(s, comp, s->buf[s->cur][comp], dense, nullptr);
}

int yb_download_field(yb_sim* s, int comp, float* dense) {
  if (!s || !dense) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (int rc = check_comp(comp)) return rc;
  YB_CU(cudaSetDevice(s->device));
  return copy_dense(s, comp, s->buf[s->cur][comp], nullptr, dense);
}

static int ensure_xfer(yb_sim* s) {
  if (s->xfer) return YB_OK;
  YB_CU(cudaStreamCreateWithFlags(&s->xfer, cudaStreamNonBlocking));
  for (cudaEvent_t& e : s->xev) YB_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return YB_OK;
}

int yb_upload_fields(yb_sim* s, const float* const* d) {
  if (!s || !d) return fail(YB_INVALID_ARGUMENT, "null argument");
  for (int c = 0; c < 6; ++c)
    if (!d[c]) return fail(YB_INVALID_ARGUMENT, "null component %d", c);
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  if (int rc = ensure_xfer(s)) return rc;
  s->q_valid = false;
  for (int c = 0; c < 6; ++c) {  // copies on the handle's stream, back to back
    int e[3];
    comp_ext(s->g, c, e);
    float* stage = s->buf[s->cur ^ 1][c];
    YB_CU(yb::copy_h2d(stage, d[c], (size_t)e[0] * e[1] * e[2] * 4, s->stream));
    YB_CU(cudaEventRecord(s->xev[c], s->stream));
    YB_CU(cudaStreamWaitEvent(s->xfer, s->xev[c], 0));  // its scatter overlaps the next copy
    YB_CU(yb::launch_scatter_dense(s->g, e, stage, s->buf[s->cur][c], s->xfer));
    YB_CU(cudaMemsetAsync(stage - yb::kGhost * s->g.plane, 0, (size_t)s->g.total * 4, s->xfer));
  }
  YB_CU(cudaEventRecord(s->xev[6], s->xfer));
  YB_CU(cudaStreamWaitEvent(s->stream, s->xev[6], 0));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_download_fields(yb_sim* s, float* const* d) {
  if (!s || !d) return fail(YB_INVALID_ARGUMENT, "null argument");
  for (int c = 0; c < 6; ++c)
    if (!d[c]) return fail(YB_INVALID_ARGUMENT, "null component %d", c);
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  if (int rc = ensure_xfer(s)) return rc;
  YB_CU(cudaEventRecord(s->xev[6], s->stream));  // the state is final
  YB_CU(cudaStreamWaitEvent(s->xfer, s->xev[6], 0));
  for (int c = 0; c < 6; ++c) {  // gathers on the side stream, each copy starts as its gather ends
    int e[3];
    comp_ext(s->g, c, e);
    float* stage = s->buf[s->cur ^ 1][c];
    YB_CU(yb::launch_gather_dense(s->g, e, s->buf[s->cur][c], stage, s->xfer));
    YB_CU(cudaEventRecord(s->xev[c], s->xfer));
    YB_CU(cudaStreamWaitEvent(s->stream, s->xev[c], 0));
    YB_CU(yb::copy_d2h(d[c], stage, (size_t)e[0] * e[1] * e[2] * 4, s->stream));
  }
  for (int c = 0; c < 6; ++c)
    YB_CU(cudaMemsetAsync(s->buf[s->cur ^ 1][c] - yb::kGhost * s->g.plane, 0, (size_t)s->g.total * 4, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

static int check_wait_error(yb_sim* s);

using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value_fn() {
  static WaitValue32Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValue32Fn>(p);
  }
  return fn;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Diagonal offsets of the skewed order for (sweeps, tile rows): diag[d] =
// (sweep, tile row) groups with 2*sweep + row < d, d = 0 .. ndiag.
static int skew_table(yb_sim* s, int nsw, int*& dev, int& cap, int& sweeps, int& tnty, int& ndiag) {
  const int nty = s->nty, nd = 2 * (nsw - 1) + nty;
  if (sweeps != nsw || tnty != nty) {
    std::vector<int> h(nd + 1, 0);
    for (int d = 0; d < nd; ++d) {
      const int lo = std::max(0, (d - nty + 2) / 2), hi = std::min(nsw - 1, d / 2);
      h[d + 1] = h[d] + std::max(0, hi - lo + 1);
    }
    if (h[nd] != nsw * nty) return fail(YB_CUDA_ERROR, "internal: skewed order covers %d of %d groups", h[nd], nsw * nty);
    if (cap < nd + 1) {
      cudaFree(dev);
      dev = nullptr;
      YB_CU(cudaMalloc(&dev, (size_t)(nd + 1) * sizeof(int)));
      cap = nd + 1;
    }
    YB_CU(cudaMemcpyAsync(dev, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    YB_CU(cudaStreamSynchronize(s->stream));
    sweeps = nsw;
    tnty = nty;
    ndiag = nd;
  }
  return YB_OK;
}

static int ensure_drain(yb_sim* s, int nsw) {
  const int nty = s->nty;
  if (int rc = skew_table(s, nsw, s->diag_dev, s->diag_cap, s->diag_sweeps, s->diag_nty, s->ndiag)) return rc;
  if (s->band_n != nty + 1) {
    cudaFree(s->band_dev);
    s->band_dev = nullptr;
    YB_CU(cudaMalloc(&s->band_dev, (size_t)(nty + 1) * sizeof(unsigned)));
    YB_CU(cudaMemsetAsync(s->band_dev, 0, (size_t)(nty + 1) * sizeof(unsigned), s->stream));
    YB_CU(cudaStreamSynchronize(s->stream));
    s->band_n = nty + 1;
    s->band_base = s->face_base = 0;
  }
  return YB_OK;
}

using Memcpy3DAsyncFn = CUresult (*)(const CUDA_MEMCPY3D*, CUstream);
static Memcpy3DAsyncFn memcpy3d_fn() {
  static Memcpy3DAsyncFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemcpy3DAsync", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Memcpy3DAsyncFn>(p);
  }
  return fn;
}

// Host <-> device copy of rows [j0, j1) of every plane of a dense e0 x e1 x e2 host array and the
// padded node box (both pitched; the copy engine, no kernel). The driver entry point with both
// memory types stated: the runtime's cudaMemcpy3DAsync spends ~150 us of host time per call.
static int copy_rows(const yb_sim* s, float* padded, float* dense, const int e[3], int j0, int j1, bool to_device,
                     cudaStream_t st, bool host_block = false) {
  CUDA_MEMCPY3D p{};
  const size_t hp = (size_t)e[0] * 4, dp = (size_t)s->g.PX * 4;
  p.srcMemoryType = to_device ? CU_MEMORYTYPE_HOST : CU_MEMORYTYPE_DEVICE;
  p.dstMemoryType = to_device ? CU_MEMORYTYPE_DEVICE : CU_MEMORYTYPE_HOST;
  if (to_device) {
    p.srcHost = dense;
    p.dstDevice = reinterpret_cast<CUdeviceptr>(padded);
  } else {
    p.srcDevice = reinterpret_cast<CUdeviceptr>(padded);
    p.dstHost = dense;
  }
  // host side: the whole dense array (rows j0.. of every plane), or — host_block — a dense block
  // of just these rows per plane (a staging chunk)
  const size_t hh = host_block ? (size_t)(j1 - j0) : (size_t)e[1], hy = host_block ? 0 : (size_t)j0;
  p.srcPitch = to_device ? hp : dp;
  p.srcHeight = to_device ? hh : (size_t)s->g.PY;
  p.dstPitch = to_device ? dp : hp;
  p.dstHeight = to_device ? (size_t)s->g.PY : hh;
  p.srcY = to_device ? hy : (size_t)j0;
  p.dstY = to_device ? (size_t)j0 : hy;
  p.WidthInBytes = hp;
  p.Height = (size_t)(j1 - j0);
  p.Depth = (size_t)e[2];
  if (CUresult r = memcpy3d_fn()(&p, reinterpret_cast<CUstream>(st)))
    return fail(YB_CUDA_ERROR, "cuMemcpy3DAsync failed (%d)", (int)r);
  return YB_OK;
}

// The readback half of a streamed run, enqueued on the transfer stream after the
// skewed launch: band ty (rows 8ty .. 8ty+7, the last band up to the face row) is
// copied once all its last-sweep row warps and all face warps have counted.
static int enqueue_band_readback(yb_sim* s, float* const* d, std::vector<cudaEvent_t>* tevp) {
  const bool trace = tevp != nullptr;
  const int nch = (s->g.nz + s->zchunk2p - 1) / s->zchunk2p;
  const unsigned per = (unsigned)(s->ntx * nch * yb::kTB2RowWarps);
  const unsigned band_need = s->band_base + per, face_need = s->face_base + s->last_grid;
  WaitValue32Fn wv = wait_value_fn();
  CUstream xs = reinterpret_cast<CUstream>(s->xfer);
  auto dptr = [&](int q) { return reinterpret_cast<CUdeviceptr>(s->band_dev + q); };
  if (CUresult r = wv(xs, dptr(s->nty), face_need, CU_STREAM_WAIT_VALUE_GEQ))
    return fail(YB_CUDA_ERROR, "cuStreamWaitValue32 failed (%d)", (int)r);
  const int fin = s->cur;  // step_tb2 flipped to the launch's final-state buffer
  for (int ty = 0; ty < s->nty; ++ty) {
    if (CUresult r = wv(xs, dptr(ty), band_need, CU_STREAM_WAIT_VALUE_GEQ))
      return fail(YB_CUDA_ERROR, "cuStreamWaitValue32 failed (%d)", (int)r);
    for (int c = 0; c < 6; ++c) {
      int e[3];
      comp_ext(s->g, c, e);
      const int j0 = ty * yb::kTB2Rows, j1 = ty == s->nty - 1 ? e[1] : std::min(j0 + yb::kTB2Rows, e[1]);
      if (j1 <= j0) continue;
      if (int rc = copy_rows(s, s->buf[fin][c], d[c], e, j0, j1, false, s->xfer)) return rc;
    }
    if (trace) YB_CU(cudaEventRecord((*tevp)[2 + ty], s->xfer));
  }
  s->band_base += per;
  s->face_base += s->last_grid;
  return YB_OK;
}

// A tile row's rows of one component as a dense block must fit a staging chunk.
static bool band_fits_staging(const yb_sim* s) {
  return (size_t)(yb::kTB2Rows + 1) * (s->g.nx + 1) * (s->g.nz + 1) * 4 <= yb::kStageBytes;
}

// The same readback into pageable buffers (the reference's own storage, array3.hpp:120): each
// (tile row, component) unit goes through the pinned staging ring of yb_xfer.cu — its pitched
// device-to-host copy lands in a chunk as a dense block (the rows x e0 of every plane), and the
// copy threads move the block's planes to their places in the caller's array while the next
// units' copies run and the rows above still sweep. Returns when all six arrays hold the state.
static int band_readback_pageable(yb_sim* s, float* const* d) {
  const int nch = (s->g.nz + s->zchunk2p - 1) / s->zchunk2p;
  const unsigned per = (unsigned)(s->ntx * nch * yb::kTB2RowWarps);
  const unsigned band_need = s->band_base + per, face_need = s->face_base + s->last_grid;
  s->band_base += per;
  s->face_base += s->last_grid;
  WaitValue32Fn wv = wait_value_fn();
  CUstream xs = reinterpret_cast<CUstream>(s->xfer);
  auto dptr = [&](int q) { return reinterpret_cast<CUdeviceptr>(s->band_dev + q); };
  struct Unit {
    int ty, c, j0, j1, e[3];
    bool first;
  };
  std::vector<Unit> units;
  for (int ty = 0; ty < s->nty; ++ty) {
    bool first = true;
    for (int c = 0; c < 6; ++c) {
      Unit u{};
      comp_ext(s->g, c, u.e);
      u.ty = ty;
      u.c = c;
      u.j0 = ty * yb::kTB2Rows;
      u.j1 = ty == s->nty - 1 ? u.e[1] : std::min(u.j0 + yb::kTB2Rows, u.e[1]);
      if (u.j1 <= u.j0) continue;
      u.first = first;
      first = false;
      units.push_back(u);
    }
  }
  std::lock_guard<std::mutex> ring(yb::stage_lock());
  YB_CU(yb::stage_init());
  if (CUresult r = wv(xs, dptr(s->nty), face_need, CU_STREAM_WAIT_VALUE_GEQ))
    return fail(YB_CUDA_ERROR, "cuStreamWaitValue32 failed (%d)", (int)r);
  const int fin = s->cur;
  auto issue = [&](size_t i) -> int {
    const Unit& u = units[i];
    const int k = (int)(i % yb::kStageChunks);
    YB_CU(yb::stage_acquire(k, s->device));
    if (u.first)
      if (CUresult r = wv(xs, dptr(u.ty), band_need, CU_STREAM_WAIT_VALUE_GEQ))
        return fail(YB_CUDA_ERROR, "cuStreamWaitValue32 failed (%d)", (int)r);
    if (int rc = copy_rows(s, s->buf[fin][u.c], static_cast<float*>(yb::stage_buf(k)), u.e, u.j0, u.j1, false, s->xfer,
                           true))
      return rc;
    YB_CU(cudaEventRecord(yb::stage_event(k), s->xfer));
    return YB_OK;
  };
  for (size_t i = 0; i < std::min<size_t>(units.size(), yb::kStageChunks); ++i)
    if (int rc = issue(i)) return rc;
  for (size_t i = 0; i < units.size(); ++i) {
    const Unit& u = units[i];
    const int k = (int)(i % yb::kStageChunks);
    YB_CU(cudaEventSynchronize(yb::stage_event(k)));
    const size_t blk = (size_t)(u.j1 - u.j0) * u.e[0];  // floats of one plane's rows
    const float* src = static_cast<const float*>(yb::stage_buf(k));
    float* dst = d[u.c];
    const int tasks = std::min(u.e[2], 16);
    yb::par_for(tasks, [&](int t) {
      const int k0 = (int)((long long)u.e[2] * t / tasks), k1 = (int)((long long)u.e[2] * (t + 1) / tasks);
      for (int kk = k0; kk < k1; ++kk)
        std::memcpy(dst + ((size_t)kk * u.e[1] + u.j0) * u.e[0], src + (size_t)kk * blk, blk * 4);
    });
    if (i + yb::kStageChunks < units.size())
      if (int rc = issue(i + yb::kStageChunks)) return rc;
  }
  return YB_OK;
}

int yb_run_to_host(yb_sim* s, int64_t nsteps, float* const* d) {
  if (!s || !d) return fail(YB_INVALID_ARGUMENT, "null argument");
  for (int c = 0; c < 6; ++c)
    if (!d[c]) return fail(YB_INVALID_ARGUMENT, "null component %d", c);
  if (nsteps < 0) return fail(YB_INVALID_ARGUMENT, "run: negative step count");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  if (s->variant != YB_VARIANT_NAIVE)
    if (int rc = prepare_fused(s)) return rc;  // sets the multi-sweep chunk (zchunk2p)
  bool pinned = true, pageable = band_fits_staging(s) && std::getenv("YB_NO_PAGEABLE_DRAIN") == nullptr;
  for (int c = 0; c < 6; ++c) {
    pinned = pinned && is_pinned(d[c]);
    pageable = pageable && yb::host_is_pageable(d[c]);
  }
  const bool stream = (pinned || pageable) && s->variant == YB_VARIANT_TB2 && s->persist && s->zchunk2p > 0 &&
                      s->probes.empty() && !s->qskip && s->g.nzg == s->g.nz && !s->peer[0].on &&
                      !s->peer[1].on && nsteps >= 4 && wait_value_fn() != nullptr && memcpy3d_fn() != nullptr &&
                      std::getenv("YB_NO_DRAIN") == nullptr;
  if (!stream) {  // the same result, read back after the run
    if (int rc = yb_advance(s, nsteps)) return rc;
    return yb_download_fields(s, d);
  }
  // the leading steps (an odd one, earlier launches of a long run) as usual,
  // then one multi-sweep launch whose tile rows stream out as they finish
  const int nsw = (int)std::min<int64_t>(nsteps / 2, 1024);
  if (int rc = yb_advance(s, nsteps - 2 * (int64_t)nsw)) return rc;
  if (int rc = prepare_fused(s)) return rc;
  // Skew only the last K sweeps: enough lead for the readback (~24 B per cell
  // over PCIe at ~52 GB/s is ~40 two-step sweeps of the kernel at ~190
  // Gcell/s, ~32 at ~160 with four coefficient arrays), at most what the tile
  // rows allow (a row leads the next by half a sweep); modelled and measured
  // with tools/drain_phases.py / tools/drain_k.sh (config 4 with the round-2 kernel: K = 32 / 40 / 48 / 56
  // -> 0.700 / 0.688 / 0.678 / 0.677 s end to end; 52 of 100).
  int K = popcount4(cell_mask(s)) > 2 ? 32 : 52;
  if (const char* e = std::getenv("YB_DRAIN_K")) K = std::atoi(e);
  K = std::max(1, std::min({K, nsw, s->nty / 2 + 1}));
  if (int rc = ensure_drain(s, K)) return rc;
  if (int rc = ensure_xfer(s)) return rc;
  // YB_DRAIN_TRACE=1 (measurement): events around the launch and after every
  // tile row's copies, printed to stderr as ms from the launch start
  const bool trace = std::getenv("YB_DRAIN_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  if (trace) {
    tev.resize(s->nty + 2);
    for (cudaEvent_t& e : tev) YB_CU(cudaEventCreate(&e));
    YB_CU(cudaEventRecord(tev[0], s->stream));
  }
  s->drain = true;
  const int rc = step_tb2(s, zfull(s), s->zchunk2p, true, nsw);
  s->drain = false;
  if (rc) return rc;
  if (trace) YB_CU(cudaEventRecord(tev[1], s->stream));
  s->step_index += 2 * nsw;
  s->steps += 2 * nsw;
  if (pinned) {
    if (int rc = enqueue_band_readback(s, d, trace ? &tev : nullptr)) return rc;
  } else {  // pageable buffers: through the staging ring, back when they hold the state
    if (int rc = band_readback_pageable(s, d)) return rc;
    if (trace)
      for (int ty = 0; ty < s->nty; ++ty) YB_CU(cudaEventRecord(tev[2 + ty], s->xfer));
  }
  s->streamed += 1;
  YB_CU(cudaEventRecord(s->xev[6], s->xfer));
  YB_CU(cudaStreamWaitEvent(s->stream, s->xev[6], 0));
  YB_CU(cudaStreamSynchronize(s->stream));
  if (trace) {
    float k = 0.f;
    YB_CU(cudaEventElapsedTime(&k, tev[0], tev[1]));
    std::fprintf(stderr, "yb_run_to_host: %d sweeps (last %d skewed), %d tile rows; kernel %.2f ms; rows done (ms):",
                 nsw, K, s->nty, k);
    for (int ty = 0; ty < s->nty; ty += std::max(1, s->nty / 16)) {
      float t = 0.f;
      YB_CU(cudaEventElapsedTime(&t, tev[0], tev[2 + ty]));
      std::fprintf(stderr, " %d:%.1f", ty, t);
    }
    float t = 0.f;
    YB_CU(cudaEventElapsedTime(&t, tev[0], tev[1 + s->nty]));
    std::fprintf(stderr, " last:%.1f\n", t);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  return check_wait_error(s);
}

using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WriteValue32Fn write_value_fn() {
  static WriteValue32Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
  }
  return fn;
}

int yb_run_streamed(yb_sim* s, int64_t nsteps, int ncoef, const int* which, const float* const* cells,
                    const float* const* in6, float* const* d) {
  if (!s || !d || (ncoef > 0 && (!which || !cells))) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (ncoef < 0 || ncoef > 4) return fail(YB_INVALID_ARGUMENT, "0 .. 4 coefficient arrays (got %d)", ncoef);
  for (int i = 0; i < ncoef; ++i) {
    if (which[i] < 0 || which[i] > 3 || !cells[i]) return fail(YB_INVALID_ARGUMENT, "bad array %d", i);
    for (int k = 0; k < i; ++k)
      if (which[k] == which[i]) return fail(YB_INVALID_ARGUMENT, "coefficient %d given twice", which[i]);
  }
  for (int c = 0; c < 6; ++c)
    if (!d[c] || (in6 && !in6[c])) return fail(YB_INVALID_ARGUMENT, "null component %d", c);
  if (nsteps < 0) return fail(YB_INVALID_ARGUMENT, "run: negative step count");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  auto plain = [&]() -> int {  // the same result, one phase after the other
    if (ncoef > 0)
      if (int rc = yb_set_cell_coeffs_n(s, ncoef, which, cells)) return rc;
    if (in6)
      if (int rc = yb_upload_fields(s, in6)) return rc;
    return yb_run_to_host(s, nsteps, d);
  };
  bool pinned = true;
  for (int c = 0; c < 6; ++c) pinned = pinned && is_pinned(d[c]) && (!in6 || is_pinned(in6[c]));
  for (int i = 0; i < ncoef; ++i) pinned = pinned && is_pinned(cells[i]);
  const int nsw = (int)(nsteps / 2);
  const bool slab = s->g.nzg != s->g.nz;
  const int nty0 = (s->g.ny + yb::kTB2Rows - 1) / yb::kTB2Rows;  // tile rows (the plan is made below)
  // Rows under 4 KB go up faster as whole arrays (measured: pitched copies of 2 KB rows reach 30 GB/s
  // against 45-52 GB/s contiguous, 4 KB rows 42 GB/s): such grids upload first, then stream the
  // readback only (YB_UP_STREAM=1 forces the streamed upload, for tests and measurement)
  const char* force = std::getenv("YB_UP_STREAM");
  const bool wide = s->g.nx >= 1024 || (force && force[0] == '1');
  // one multi-sweep launch carries the whole run: an even step count, at most 2048 steps,
  // enough sweeps and tile rows to skew both ends; every host array page-locked
  if (!(pinned && wide && (ncoef > 0 || in6) && s->variant == YB_VARIANT_TB2 && s->persist && s->probes.empty() && !s->qskip &&
        !slab && !s->peer[0].on && !s->peer[1].on && nsteps % 2 == 0 && nsw >= 4 && nsw <= 1024 && nty0 >= 4 &&
        wait_value_fn() && write_value_fn() && memcpy3d_fn() && std::getenv("YB_NO_DRAIN") == nullptr &&
        std::getenv("YB_NO_UPSTREAM") == nullptr))
  {
    if (std::getenv("YB_STREAM_DEBUG"))
      std::fprintf(stderr,
                   "yb_run_streamed: phase by phase (pinned %d, wide %d, arrays %d, variant %d, persist %d, probes %d, qskip %d, "
                   "slab %d, nsteps %lld, tile rows %d, wait fn %d, write fn %d)\n",
                   (int)pinned, (int)wide, ncoef + (in6 ? 6 : 0), s->variant, (int)s->persist, (int)s->probes.size(), (int)s->qskip,
                   (int)slab, (long long)nsteps, nty0, wait_value_fn() != nullptr, write_value_fn() != nullptr);
    return plain();
  }
  // The arrays as given, zero outside the cell box (no uniformity compression: a uniform array
  // multiplies by the same values the scalar would); their clamped duplicates are filled after the run.
  for (int i = 0; i < ncoef; ++i) {
    const int w = which[i];
    if (!s->cell[w]) {
      float* p = nullptr;
      YB_CU(cudaMalloc(&p, (size_t)s->g.total * 4));
      s->cell[w] = p + yb::kGhost * s->g.plane;
      s->dev_bytes += (size_t)s->g.total * 4;
    }
    YB_CU(cudaMemsetAsync(s->cell[w] - yb::kGhost * s->g.plane, 0, (size_t)s->g.total * 4, s->stream));
    if (w == YB_CB) s->cb_uniform = false;
    if (w == YB_DB) s->db_uniform = false;
  }
  if (ncoef > 0) s->tm_valid = false;
  s->q_valid = false;
  if (int rc = prepare_fused(s)) return rc;
  if (s->zchunk2p <= 0 || s->nty != nty0) return plain();
  // Tail skew as yb_run_to_host. Head skew: as many sweeps as the upload lasts (they trail it tile
  // row by tile row; ~45 GB/s of pitched copies against ~185 / ~155 Gcell/s sweeps) plus two —
  // skewed sweeps are ~15% slower (a tile row's y-halo rows miss L2), so no deeper than needed.
  const bool heavy = popcount4(cell_mask(s)) > 2;
  int K = heavy ? 32 : 52;
  if (const char* e = std::getenv("YB_DRAIN_K")) K = std::atoi(e);
  const double cells1 = (double)s->g.nx * s->g.ny * s->g.nz;
  const double up_s = (ncoef * cells1 + (in6 ? 6.0 * cells1 : 0.0)) * 4.0 / 45e9;
  int Kh = (int)std::ceil(up_s / (2.0 * cells1 / (heavy ? 155e9 : 185e9))) + 2;
  if (const char* e = std::getenv("YB_UP_K")) Kh = std::atoi(e);
  const int kmax = s->nty / 2 + 1;
  K = std::max(1, std::min(K, kmax));
  Kh = std::max(1, std::min(Kh, kmax));
  if (K + Kh > nsw) {  // a short run: share the sweeps in proportion
    Kh = std::max(1, std::min(nsw - 1, (int)((long long)nsw * Kh / (K + Kh))));
    K = nsw - Kh;
  }
  if (int rc = ensure_drain(s, K)) return rc;
  if (int rc = skew_table(s, Kh, s->diagh_dev, s->diagh_cap, s->diagh_sweeps, s->diagh_nty, s->ndiagh)) return rc;
  if (int rc = ensure_xfer(s)) return rc;
  if (s->upband_n != s->nty) {
    cudaFree(s->upband_dev);
    s->upband_dev = nullptr;
    YB_CU(cudaMalloc(&s->upband_dev, (size_t)s->nty * sizeof(unsigned)));
    YB_CU(cudaMemsetAsync(s->upband_dev, 0, (size_t)s->nty * sizeof(unsigned), s->stream));
    s->upband_n = s->nty;
    s->up_base = 0;
  }
  // the copies: tile row by tile row on the transfer stream, each row's word written behind them
  YB_CU(cudaEventRecord(s->xev[6], s->stream));  // the zeroed arrays; earlier work on the state
  YB_CU(cudaStreamWaitEvent(s->xfer, s->xev[6], 0));
  WriteValue32Fn wr = write_value_fn();
  CUstream xs = reinterpret_cast<CUstream>(s->xfer);
  // YB_DRAIN_TRACE=1 (measurement): events after every tile row's copies (both directions) and
  // around the launch, printed to stderr as ms from the first copy
  const bool trace = std::getenv("YB_DRAIN_TRACE") != nullptr;
  std::vector<cudaEvent_t> uev, tev;
  if (trace) {
    uev.resize(s->nty + 1);
    tev.resize(s->nty + 2);
    for (cudaEvent_t& e : uev) YB_CU(cudaEventCreate(&e));
    for (cudaEvent_t& e : tev) YB_CU(cudaEventCreate(&e));
    YB_CU(cudaEventRecord(uev[s->nty], s->xfer));
  }
  const unsigned need = s->up_base + 1;
  const int ce[3] = {s->g.nx, s->g.ny, s->g.nz};
  if (trace) YB_CU(cudaEventRecord(tev[0], s->stream));
  s->drain = true;
  s->upstream = true;
  const int cur0 = s->cur;  // the launch's input state (step_tb2 flips to the final-state buffer)
  const int rc = step_tb2(s, zfull(s), s->zchunk2p, true, nsw);
  s->drain = false;
  s->upstream = false;
  s->up_base = need;
  if (rc) return rc;
  // the launch is in flight (its first-sweep items poll the row words): now the copies. Should one
  // fail to enqueue, every row word is released (the run's result is then undefined, the call
  // returns the error) so that the launch does not spin until its deadline.
  auto release_rows = [&](int rc) {
    std::vector<unsigned> w((size_t)s->nty, need);
    cudaMemcpyAsync(s->upband_dev, w.data(), w.size() * sizeof(unsigned), cudaMemcpyHostToDevice, s->xfer);
    cudaStreamSynchronize(s->xfer);
    cudaStreamSynchronize(s->stream);
    return rc;
  };
  // (one copy stream: the arrays alternating over two streams measured no faster)
  for (int ty = 0; ty < s->nty; ++ty) {
    const int j0 = ty * yb::kTB2Rows;
    const bool last = ty == s->nty - 1;
    for (int i = 0; i < ncoef; ++i) {
      const int j1 = last ? ce[1] : std::min(j0 + yb::kTB2Rows, ce[1]);
      if (j1 > j0)
        if (int rc = copy_rows(s, s->cell[which[i]], const_cast<float*>(cells[i]), ce, j0, j1, true, s->xfer))
          return release_rows(rc);
    }
    if (in6)
      for (int c = 0; c < 6; ++c) {
        int e[3];
        comp_ext(s->g, c, e);
        const int j1 = last ? e[1] : std::min(j0 + yb::kTB2Rows, e[1]);
        if (j1 > j0)
          if (int rc = copy_rows(s, s->buf[cur0][c], const_cast<float*>(in6[c]), e, j0, j1, true, s->xfer))
            return release_rows(rc);
      }
    if (CUresult r = wr(xs, reinterpret_cast<CUdeviceptr>(s->upband_dev + ty), need, 0))
      return release_rows(fail(YB_CUDA_ERROR, "cuStreamWriteValue32 failed (%d)", (int)r));
    if (trace) YB_CU(cudaEventRecord(uev[ty], s->xfer));
  }
  s->step_index += 2 * nsw;
  s->steps += 2 * nsw;
  for (int i = 0; i < ncoef; ++i)  // the arrays' clamped duplicates (other kernels read them), behind the run
    YB_CU(yb::launch_clamp_fill(s->g, s->cell[which[i]], 0, s->g.nz - 1, s->stream));
  if (trace) YB_CU(cudaEventRecord(tev[1], s->stream));
  if (int rc2 = enqueue_band_readback(s, d, trace ? &tev : nullptr)) return rc2;
  s->streamed += 1;
  s->streamed_up += 1;
  YB_CU(cudaEventRecord(s->xev[6], s->xfer));
  YB_CU(cudaStreamWaitEvent(s->stream, s->xev[6], 0));
  YB_CU(cudaStreamSynchronize(s->stream));
  if (trace) {
    auto ms = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, uev[s->nty], e);
      return t;
    };
    std::fprintf(stderr, "yb_run_streamed: %d sweeps (first %d, last %d skewed), %d tile rows; launch %.1f .. %.1f ms; rows up (ms):",
                 nsw, Kh, K, s->nty, ms(tev[0]), ms(tev[1]));
    const int st = std::max(1, s->nty / 8);
    for (int ty = 0; ty < s->nty; ty += st) std::fprintf(stderr, " %d:%.1f", ty, ms(uev[ty]));
    std::fprintf(stderr, " last:%.1f; rows down (ms):", ms(uev[s->nty - 1]));
    for (int ty = 0; ty < s->nty; ty += st) std::fprintf(stderr, " %d:%.1f", ty, ms(tev[2 + ty]));
    std::fprintf(stderr, " last:%.1f\n", ms(tev[1 + s->nty]));
    for (cudaEvent_t e : uev) cudaEventDestroy(e);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  return check_wait_error(s);
}

int yb_zero_fields(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  for (int c = 0; c < 6; ++c)
    YB_CU(cudaMemsetAsync(s->buf[s->cur][c] - yb::kGhost * s->g.plane, 0, (size_t)s->g.total * 4, s->stream));
  s->step_index = 0;
  s->q_valid = false;
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_fill_fields(yb_sim* s, uint64_t seed) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  YB_CU(cudaSetDevice(s->device));
  YB_CU(yb::launch_fill_fields(s->g, fields_of(s, s->cur), seed, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  s->q_valid = false;
  return YB_OK;
}

int yb_set_step_index(yb_sim* s, int64_t v) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (v < 0) return fail(YB_INVALID_ARGUMENT, "negative step index");
  s->step_index = v;
  return YB_OK;
}

int yb_get_step_index(yb_sim* s, int64_t* v) {
  if (!s || !v) return fail(YB_INVALID_ARGUMENT, "null argument");
  *v = s->step_index;
  return YB_OK;
}

int yb_add_source(yb_sim* s, int comp, int i, int j, int k, const float* table, int64_t n) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (comp < 0 || comp > 2) return fail(YB_INVALID_ARGUMENT, "SourceSpec: component must be electric");
  if (n < 0 || (n > 0 && !table)) return fail(YB_INVALID_ARGUMENT, "SourceSpec: bad table");
  if ((int)s->sources.size() >= YB_MAX_SOURCES)
    return fail(YB_INVALID_ARGUMENT, "at most %d sources", YB_MAX_SOURCES);
  // strictly interior (source.hpp:43-55): node axes 1..n-1, the half axis 1..n-2
  const int idx[3] = {i, j, k};
  const int ns[3] = {s->g.nx, s->g.ny, s->g.nzg};
  for (int a = 0; a < 3; ++a) {
    const bool node = a != comp;
    const int lo = 1, hi = node ? ns[a] : ns[a] - 1;
    if (idx[a] < lo || idx[a] >= hi) return fail(YB_INVALID_ARGUMENT, "SourceSpec: position not interior");
  }
  Src q{comp, i, j, k, std::vector<float>(table, table + n)};
  s->sources.push_back(std::move(q));
  return YB_OK;
}

int yb_clear_sources(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  s->sources.clear();
  return YB_OK;
}

static bool probe_fires(const yb_sim* s, int64_t step) {
  for (const Probe& p : s->probes)
    if (step % p.stride == 0) return true;
  return false;
}

// Records every probe firing at the current step_index (on the device).
static int sample_probes_dev(yb_sim* s) {
  yb::ProbeArgs pa{};
  for (size_t q = 0; q < s->probes.size(); ++q) {
    const Probe& p = s->probes[q];
    if (s->step_index % p.stride) continue;
    pa.comp[pa.n] = p.comp;
    pa.off[pa.n] = ((long long)p.k * s->g.PY + p.j) * s->g.PX + p.i;
    ++pa.n;
    s->probe_meta.push_back({s->step_index, (int)q});
  }
  if (!pa.n) return YB_OK;
  const size_t need = s->probe_meta.size();
  if (need > s->probe_cap) {  // grow (rare): copy the recorded values over
    size_t cap = std::max<size_t>(1024, 2 * s->probe_cap);
    while (cap < need) cap *= 2;
    float* nb = nullptr;
    YB_CU(cudaMalloc(&nb, cap * sizeof(float)));
    if (s->probe_dev) {
      YB_CU(cudaMemcpyAsync(nb, s->probe_dev, (need - pa.n) * sizeof(float), cudaMemcpyDeviceToDevice,
                            s->stream));
      YB_CU(cudaStreamSynchronize(s->stream));
      YB_CU(cudaFree(s->probe_dev));
    }
    s->probe_dev = nb;
    s->probe_cap = cap;
  }
  YB_CU(yb::launch_probes(fields_of(s, s->cur), pa, s->probe_dev + (need - pa.n), s->stream));
  s->launches += 1;
  return YB_OK;
}

int yb_advance(yb_sim* s, int64_t nsteps) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (nsteps < 0) return fail(YB_INVALID_ARGUMENT, "run: negative step count");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end)");
  YB_CU(cudaSetDevice(s->device));
  if (s->variant != YB_VARIANT_NAIVE) {
    if (int rc = prepare_fused(s)) return rc;
    if (int rc = qmap_refresh(s)) return rc;
  }
  const bool probes = !s->probes.empty();
  for (int64_t t = 0; t < nsteps;) {
    // four steps per launch (TB4) unless a probe wants a level in between
    if (s->variant == YB_VARIANT_TB4 && t + 4 <= nsteps &&
        !(probes && (probe_fires(s, s->step_index + 1) || probe_fires(s, s->step_index + 2) ||
                     probe_fires(s, s->step_index + 3)))) {
      if (int rc = step_tb4(s)) return rc;
      s->step_index += 4;
      s->steps += 4;
      t += 4;
      if (probes && probe_fires(s, s->step_index))
        if (int rc = sample_probes_dev(s)) return rc;
      continue;
    }
    if (s->qskip && !s->q_valid)
      if (int rc = qmap_refresh(s)) return rc;
    // several two-step sweeps in one launch (single domain, no probes, no
    // quiescent skip): items of the next sweep start as their neighbourhood
    // finishes, so no launch gap or wave tail separates the sweeps
    if (s->variant == YB_VARIANT_TB2 && s->persist && s->zchunk2p > 0 && !probes && !s->qskip &&
        s->g.nzg == s->g.nz && nsteps - t >= 4) {
      const int nsw = (int)std::min<int64_t>((nsteps - t) / 2, 1024);
      if (int rc = step_tb2(s, zfull(s), s->zchunk2p, true, nsw)) return rc;
      s->step_index += 2 * nsw;
      s->steps += 2 * nsw;
      t += 2 * nsw;
      continue;
    }
    // two steps per launch unless a probe wants the level in between
    if ((s->variant == YB_VARIANT_TB2 || s->variant == YB_VARIANT_TB4) && t + 2 <= nsteps &&
        !(probes && probe_fires(s, s->step_index + 1))) {
      if (int rc = step_tb2(s, zfull(s), s->zchunk2, true)) return rc;
      s->step_index += 2;
      s->steps += 2;
      t += 2;
    } else {
      const int rc = s->variant == YB_VARIANT_NAIVE ? step_naive(s) : step_fused(s, zfull(s), s->zchunk, true);
      if (rc) return rc;
      ++s->step_index;
      ++s->steps;
      ++t;
    }
    if (probes && probe_fires(s, s->step_index))
      if (int rc = sample_probes_dev(s)) return rc;
  }
  return YB_OK;
}

int yb_snapshot_h(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  YB_CU(cudaSetDevice(s->device));
  const size_t n = (size_t)s->g.plane * (s->g.nz + 1);
  for (int c = 0; c < 3; ++c) {
    if (!s->snap_h[c]) {
      YB_CU(cudaMalloc(&s->snap_h[c], n * sizeof(float)));
      s->dev_bytes += n * sizeof(float);
    }
    YB_CU(cudaMemcpyAsync(s->snap_h[c], s->buf[s->cur][3 + c], n * sizeof(float), cudaMemcpyDeviceToDevice,
                          s->stream));
  }
  s->have_snap = true;
  return YB_OK;
}

int yb_total_energy(yb_sim* s, const double* dx, const double* dy, const double* dz, double* energy) {
  if (!s || !energy) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (!s->have_snap) return fail(YB_INVALID_ARGUMENT, "total_energy: no H snapshot (call yb_snapshot_h first)");
  YB_CU(cudaSetDevice(s->device));
  const Geo& g = s->g;
  // dual spacing at node i: half-sum of the adjacent cells, halved at the ends
  // (dual_spacing, fields.hpp:86-93); primal spacing at cell i: d[i].
  std::vector<double> w;
  auto axis = [&](const double* d, int n, int off, int nglob, int count) {
    auto at = [&](int q) { return d ? d[q] : 1.0; };
    for (int q = off; q <= off + count; ++q)
      w.push_back(q == 0 ? 0.5 * at(0) : (q == nglob ? 0.5 * at(nglob - 1) : 0.5 * (at(q - 1) + at(q))));
    for (int q = off; q < off + count; ++q) w.push_back(at(q));
  };
  axis(dx, g.nx, 0, g.nx, g.nx);
  axis(dy, g.ny, 0, g.ny, g.ny);
  axis(dz, g.nzg, g.zoff, g.nzg, g.nz);
  const size_t nw = w.size(), np = 6 * yb::kEnergyBlocks;
  if (!s->energy_dev) YB_CU(cudaMalloc(&s->energy_dev, (nw + np + 1) * sizeof(double)));
  double* wd = s->energy_dev;
  YB_CU(cudaMemcpyAsync(wd, w.data(), nw * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  const float* prev[3] = {s->snap_h[0], s->snap_h[1], s->snap_h[2]};
  YB_CU(yb::launch_energy(g, fields_of(s, s->cur), prev, wd, wd + nw, wd + nw + np, s->stream));
  s->launches += 2;
  YB_CU(cudaMemcpyAsync(energy, wd + nw + np, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_advance_begin(yb_sim* s, int64_t nsteps) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is already in flight");
  if (s->variant == YB_VARIANT_NAIVE) return fail(YB_INVALID_ARGUMENT, "split sweeps need the FUSED or TB2 variant");
  if (nsteps < 1 || nsteps > 2 || (nsteps == 2 && s->variant != YB_VARIANT_TB2 && s->variant != YB_VARIANT_TB4))
    return fail(YB_INVALID_ARGUMENT, "split sweep: 1 step (FUSED / TB2) or 2 steps (TB2)");
  if (!s->probes.empty()) return fail(YB_INVALID_ARGUMENT, "split sweeps do not sample probes");
  YB_CU(cudaSetDevice(s->device));
  if (int rc = prepare_fused(s)) return rc;
  if (int rc = qmap_refresh(s)) return rc;
  const int b = (int)nsteps, nz = s->g.nz;
  s->pending_full = nz <= 2 * b + 1;  // no interior worth a launch: one whole sweep
  const ZPart z = s->pending_full ? zfull(s) : ZPart{0, b, nz - b, nz};
  const int zc = s->pending_full ? (nsteps == 2 ? s->zchunk2 : s->zchunk) : b;
  if (!s->side) {
    YB_CU(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
    YB_CU(cudaEventCreateWithFlags(&s->ev_pre, cudaEventDisableTiming));
    YB_CU(cudaEventCreateWithFlags(&s->ev_int, cudaEventDisableTiming));
    YB_CU(cudaMalloc(&s->sched2, sizeof(unsigned long long)));
    YB_CU(cudaMemsetAsync(s->sched2, 0, sizeof(unsigned long long), s->stream));
    s->sched2_base = 0;
  }
  YB_CU(cudaEventRecord(s->ev_pre, s->stream));  // the state the interior launch will read is complete
  if (int rc = nsteps == 2 ? step_tb2(s, z, zc, false) : step_fused(s, z, zc, false)) return rc;
  s->pending = (int)nsteps;
  return YB_OK;
}

int yb_advance_end(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (!s->pending) return fail(YB_INVALID_ARGUMENT, "no split sweep in flight (yb_advance_begin)");
  YB_CU(cudaSetDevice(s->device));
  const int n = s->pending, nz = s->g.nz;
  if (!s->pending_full) {
    // the interior on the side stream, concurrent with the boundary launch and
    // whatever the caller enqueued since (pack, transfers); the handle's
    // stream then waits for it
    const ZPart z{n, nz - n, nz - n, nz - n};
    YB_CU(cudaStreamWaitEvent(s->side, s->ev_pre, 0));
    s->on_side = true;
    const int rc = n == 2 ? step_tb2(s, z, s->zchunk2, false) : step_fused(s, z, s->zchunk, false);
    s->on_side = false;
    if (rc) return rc;
    YB_CU(cudaEventRecord(s->ev_int, s->side));
    YB_CU(cudaStreamWaitEvent(s->stream, s->ev_int, 0));
  }
  s->cur ^= 1;
  s->step_index += n;
  s->steps += n;
  s->pending = 0;
  return YB_OK;
}

int yb_set_probes(yb_sim* s, int n, const int* comp, const int* i, const int* j, const int* k,
                  const int* stride) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (n < 0 || n > YB_MAX_PROBES) return fail(YB_INVALID_ARGUMENT, "at most %d probes", YB_MAX_PROBES);
  if (n > 0 && (!comp || !i || !j || !k || !stride)) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (n > 0 && s->g.nzg != s->g.nz) return fail(YB_INVALID_ARGUMENT, "probes: single-domain handles only");
  std::vector<Probe> ps;
  for (int q = 0; q < n; ++q) {  // ProbeSpec::validate (probe.hpp:21-25)
    if (stride[q] < 1) return fail(YB_INVALID_ARGUMENT, "ProbeSpec: stride must be >= 1");
    if (int rc = check_comp(comp[q])) return rc;
    int e[3];
    comp_ext(s->g, comp[q], e);
    if (i[q] < 0 || i[q] >= e[0] || j[q] < 0 || j[q] >= e[1] || k[q] < 0 || k[q] >= e[2])
      return fail(YB_INVALID_ARGUMENT, "ProbeSpec: position outside grid");
    ps.push_back({comp[q], i[q], j[q], k[q], stride[q]});
  }
  s->probes = ps;
  return YB_OK;
}

int yb_read_probes(yb_sim* s, int64_t* steps, int* probe, float* values, int64_t capacity,
                   int64_t* count) {
  if (!s || !count || capacity < 0) return fail(YB_INVALID_ARGUMENT, "bad argument");
  const int64_t n = std::min<int64_t>(capacity, (int64_t)s->probe_meta.size());
  *count = n;
  if (n == 0) return YB_OK;
  if (!steps || !probe || !values) return fail(YB_INVALID_ARGUMENT, "null argument");
  YB_CU(cudaSetDevice(s->device));
  YB_CU(cudaMemcpyAsync(values, s->probe_dev, n * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  for (int64_t q = 0; q < n; ++q) {
    steps[q] = s->probe_meta[q].first;
    probe[q] = s->probe_meta[q].second;
  }
  const int64_t rest = (int64_t)s->probe_meta.size() - n;
  if (rest > 0) {  // keep the unread tail at the front
    YB_CU(cudaMemcpyAsync(s->probe_dev, s->probe_dev + n, rest * sizeof(float), cudaMemcpyDeviceToDevice,
                          s->stream));
    YB_CU(cudaStreamSynchronize(s->stream));
  }
  s->probe_meta.erase(s->probe_meta.begin(), s->probe_meta.begin() + n);
  return YB_OK;
}

// Reports (and clears) the record of a spin wait that passed its deadline.
static int check_wait_error(yb_sim* s) {
  int r[8] = {};
  YB_CU(cudaMemcpy(r, s->werr, sizeof r, cudaMemcpyDeviceToHost));
  if (r[0] == 0) return YB_OK;
  YB_CU(cudaMemset(s->werr, 0, sizeof r));
  const double ms = (double)s->wait_ns * 1e-6;
  if (r[0] == yb::WAIT_DEP) {
    const int T = s->ntx * s->nty, ch = r[1] / T, tile = r[1] % T;
    return fail(YB_RUNTIME_ERROR,
                "multi-sweep launch: work item %d (tile x=%d y=%d, z-chunk %d) of sweep %d waited more than "
                "%.0f ms for its neighbourhood (completion count %u, needed %u)",
                r[1], tile % s->ntx, tile / s->ntx, ch, r[2], ms, (unsigned)r[3], (unsigned)r[4]);
  }
  const char* side = r[2] == 0 ? "below" : "above";
  if (r[0] == yb::WAIT_PEER_KERNEL)
    return fail(YB_RUNTIME_ERROR,
                "peer-store sweep: boundary work item %d waited more than %.0f ms for the slab %s "
                "(flag %u, needed %u: that neighbour never signalled)",
                r[1], ms, side, (unsigned)r[3], (unsigned)r[4]);
  return fail(YB_RUNTIME_ERROR,
              "peer halo wait: more than %.0f ms for the slab %s (flag %u, needed %u: that neighbour never signalled)",
              ms, side, (unsigned)r[3], (unsigned)r[4]);
}

int yb_synchronize(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  YB_CU(cudaSetDevice(s->device));
  YB_CU(cudaStreamSynchronize(s->stream));
  if (s->peer_stream) YB_CU(cudaStreamSynchronize(s->peer_stream));
  if (int rc = check_wait_error(s)) return rc;
  return collect_timers(s);
}

int yb_advance_timed(yb_sim* s, int64_t nsteps, float* ms) {
  if (!s || !ms) return fail(YB_INVALID_ARGUMENT, "null argument");
  YB_CU(cudaSetDevice(s->device));
  if (s->variant != YB_VARIANT_NAIVE)
    if (int rc = prepare_fused(s)) return rc;
  cudaEvent_t a, b;
  YB_CU(cudaEventCreate(&a));
  YB_CU(cudaEventCreate(&b));
  YB_CU(cudaEventRecord(a, s->stream));
  int rc = yb_advance(s, nsteps);
  if (rc == YB_OK) {
    YB_CU(cudaEventRecord(b, s->stream));
    YB_CU(cudaEventSynchronize(b));
    YB_CU(cudaEventElapsedTime(ms, a, b));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return rc;
}

static int check_box(const yb_sim* s, const int* box, int out[6]) {
  const int full[6] = {0, s->g.nx + 1, 0, s->g.ny + 1, 0, s->g.nz + 1};
  if (!box) {
    std::memcpy(out, full, sizeof full);
    return YB_OK;
  }
  const bool empty = box[1] <= box[0] || box[3] <= box[2] || box[5] <= box[4];
  if (!empty && (box[0] < 0 || box[1] > full[1] || box[2] < 0 || box[3] > full[3] || box[4] < 0 ||
                 box[5] > full[5]))
    return fail(YB_OUT_OF_RANGE, "range out of bounds");
  std::memcpy(out, box, 6 * sizeof(int));
  return YB_OK;
}

static bool slab_mode(const yb_sim* s) { return s->g.nzg != s->g.nz; }

int yb_apply_ampere_range(yb_sim* s, const int* box) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (slab_mode(s)) return fail(YB_INVALID_ARGUMENT, "range ops act on a whole domain, not a z-slab");
  int b[6];
  if (int rc = check_box(s, box, b)) return fail(rc, "apply_ampere_range: range out of bounds");
  YB_CU(cudaSetDevice(s->device));
  s->q_valid = false;
  YB_CU(yb::launch_naive_ampere(s->g, fields_of(s, s->cur), coef_args(s), b, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_apply_faraday_range(yb_sim* s, const int* box) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (slab_mode(s)) return fail(YB_INVALID_ARGUMENT, "range ops act on a whole domain, not a z-slab");
  int b[6];
  if (int rc = check_box(s, box, b)) return fail(rc, "apply_faraday_range: range out of bounds");
  YB_CU(cudaSetDevice(s->device));
  s->q_valid = false;
  YB_CU(yb::launch_naive_faraday(s->g, fields_of(s, s->cur), coef_args(s), b, s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_apply_pec_boundary(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight (yb_advance_end first)");
  if (slab_mode(s)) return fail(YB_INVALID_ARGUMENT, "range ops act on a whole domain, not a z-slab");
  YB_CU(cudaSetDevice(s->device));
  s->q_valid = false;
  YB_CU(yb::launch_naive_pec(s->g, fields_of(s, s->cur), s->stream));
  YB_CU(cudaStreamSynchronize(s->stream));
  return YB_OK;
}

int yb_field_digest(yb_sim* s, uint64_t* out) {
  if (!s || !out) return fail(YB_INVALID_ARGUMENT, "null argument");
  uint64_t h = 1469598103934665603ull;
  std::vector<float> host;
  for (int c = 0; c < 6; ++c) {
    int e[3];
    comp_ext(s->g, c, e);
    host.resize((size_t)e[0] * e[1] * e[2]);
    if (int rc = yb_download_field(s, c, host.data())) return rc;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(host.data());
    for (size_t q = 0; q < host.size() * 4; ++q) {
      h ^= b[q];
      h *= 1099511628211ull;
    }
  }
  *out = h;
  return YB_OK;
}

// z-slab halo planes (see include/yeeb200.h). Depth d = 1 (one-step
// sweeps) or 2 (two-step sweeps). Down-send: my planes 0..d-1, all six
// components (-> the slab below's ghost planes nz..nz+d-1). Up-send: my planes
// nz-d+1..nz-1 all six, plane nz-d hx, hy (-> the slab above's ghost planes
// -d+1..-1 and -d). Planes are contiguous (PX*PY floats): one device copy each.
static int halo_depth(const yb_sim* s) { return s->variant == YB_VARIANT_FUSED || s->variant == YB_VARIANT_NAIVE ? 1 : 2; }
static int halo_planes(const yb_sim* s, bool down) {
  const int d = halo_depth(s);
  return down ? 6 * d : 6 * (d - 1) + 2;
}

int yb_halo_bytes(yb_sim* s, int side, int receive, size_t* bytes) {
  if (!s || !bytes || side < 0 || side > 1) return fail(YB_INVALID_ARGUMENT, "bad argument");
  // side 0 sends down / receives up-data; side 1 sends up / receives down-data
  const bool down = (side == 0) != (receive != 0);
  *bytes = (size_t)halo_planes(s, down) * s->g.plane * sizeof(float);
  return YB_OK;
}

static int halo_copy(yb_sim* s, int side, char* ext, bool pack) {
  YB_CU(cudaSetDevice(s->device));
  const size_t pb = (size_t)s->g.plane * sizeof(float);
  const int d = halo_depth(s), nz = s->g.nz;
  // (component, local plane) list in buffer order
  int comp[12], plane[12], n = 0;
  const bool down_data = (side == 0) == pack;  // planes 0.. of the slab above
  if (down_data) {
    const int base = pack ? 0 : nz;  // my planes 0..d-1, or my ghosts nz..nz+d-1
    for (int q = 0; q < d; ++q)
      for (int c = 0; c < 6; ++c) comp[n] = c, plane[n++] = base + q;
  } else {
    const int base = pack ? nz - d : -d;  // my planes nz-d..nz-1, or my ghosts -d..-1
    comp[n] = YB_HX, plane[n++] = base;
    comp[n] = YB_HY, plane[n++] = base;
    for (int q = 1; q < d; ++q)
      for (int c = 0; c < 6; ++c) comp[n] = c, plane[n++] = base + q;
  }
  const int b = s->pending && pack ? s->cur ^ 1 : s->cur;  // a split sweep's new boundary planes
  cudaPointerAttributes at{};
  const bool dev_ext = cudaPointerGetAttributes(&at, ext) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
                       at.device == s->device;
  cudaGetLastError();  // clear a "not a device pointer" status
  if (dev_ext) {  // one copy kernel for every plane
    yb::HaloList l{};
    for (int q = 0; q < n; ++q) l.plane[q] = s->buf[b][comp[q]] + (long long)plane[q] * s->g.plane;
    l.n = n;
    YB_CU(yb::launch_halo_copy(s->g, l, reinterpret_cast<float*>(ext), pack, s->stream));
  } else {
    for (int q = 0; q < n; ++q) {
      float* dev = s->buf[b][comp[q]] + (long long)plane[q] * s->g.plane;
      if (pack)
        YB_CU(cudaMemcpyAsync(ext + q * pb, dev, pb, cudaMemcpyDefault, s->stream));
      else
        YB_CU(cudaMemcpyAsync(dev, ext + q * pb, pb, cudaMemcpyDefault, s->stream));
    }
  }
  if (s->stream == s->own_stream) YB_CU(cudaStreamSynchronize(s->stream));  // else stream-ordered
  return YB_OK;
}

int yb_halo_pack(yb_sim* s, int side, void* dst) {
  if (!s || !dst || side < 0 || side > 1) return fail(YB_INVALID_ARGUMENT, "bad argument");
  return halo_copy(s, side, static_cast<char*>(dst), true);
}

int yb_halo_unpack(yb_sim* s, int side, const void* src) {
  if (!s || !src || side < 0 || side > 1) return fail(YB_INVALID_ARGUMENT, "bad argument");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "halo_unpack during a split sweep (after yb_advance_end)");
  if (int rc = halo_copy(s, side, const_cast<char*>(static_cast<const char*>(src)), false)) return rc;
  if (s->qskip && s->q_valid) {  // the ghost planes just written: mark the nonzero tile-planes
    const int d = halo_depth(s);
    const int k0 = side == 0 ? -d : s->g.nz, k1 = side == 0 ? -1 : s->g.nz + d - 1;
    YB_CU(yb::launch_qscan(s->g, fields_of(s, 0), fields_of(s, 1), qmap_of(s), k0, k1, s->stream));
  }
  return YB_OK;
}

// ------------------------------------------------------------ peer halos
static int ensure_pflags(yb_sim* s) {
  if (s->pflags) return YB_OK;
  YB_CU(cudaSetDevice(s->device));
  YB_CU(cudaMalloc(&s->pflags, 8 * sizeof(unsigned)));  // + [4], [5]: boundary-item counters
  YB_CU(cudaMemset(s->pflags, 0, 8 * sizeof(unsigned)));
  return YB_OK;
}

size_t yb_peer_handle_bytes(void) { return 13 * sizeof(cudaIpcMemHandle_t); }

int yb_peer_export(yb_sim* s, void* out) {
  if (!s || !out) return fail(YB_INVALID_ARGUMENT, "null argument");
  if (int rc = ensure_pflags(s)) return rc;
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(out);
  for (int b = 0; b < 2; ++b)
    for (int c = 0; c < 6; ++c) YB_CU(cudaIpcGetMemHandle(&h[b * 6 + c], s->buf[b][c] - yb::kGhost * s->g.plane));
  YB_CU(cudaIpcGetMemHandle(&h[12], s->pflags));
  return YB_OK;
}

static int check_peer_args(yb_sim* s, int side, int peer_nz) {
  if (!s || side < 0 || side > 1 || peer_nz < 1) return fail(YB_INVALID_ARGUMENT, "bad argument");
  if (s->g.nzg == s->g.nz) return fail(YB_INVALID_ARGUMENT, "peer halos need a z-slab handle");
  if ((side == 0 && at_bottom(s->g)) || (side == 1 && at_top(s->g)))
    return fail(YB_INVALID_ARGUMENT, "no neighbour on that side (global boundary)");
  return ensure_pflags(s);
}

int yb_peer_open(yb_sim* s, int side, const void* handles, int peer_nz) {
  if (!handles) return fail(YB_INVALID_ARGUMENT, "null handles");
  if (int rc = check_peer_args(s, side, peer_nz)) return rc;
  YB_CU(cudaSetDevice(s->device));
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  PeerSide& ps = s->peer[side];
  for (int q = 0; q < 13; ++q) {
    void* p = nullptr;
    YB_CU(cudaIpcOpenMemHandle(&p, h[q], cudaIpcMemLazyEnablePeerAccess));
    ps.ipc.push_back(p);
    if (q < 12)
      ps.buf[q / 6][q % 6] = static_cast<float*>(p) + yb::kGhost * s->g.plane;  // same PX, PY by construction
    else
      ps.flags = static_cast<unsigned*>(p);
  }
  ps.nz = peer_nz;
  ps.on = true;
  return YB_OK;
}

int yb_peer_link(yb_sim* s, int side, yb_sim* other) {
  if (!other) return fail(YB_INVALID_ARGUMENT, "null peer");
  if (int rc = check_peer_args(s, side, other->g.nz)) return rc;
  if (int rc = ensure_pflags(other)) return rc;
  if (other->g.nx != s->g.nx || other->g.ny != s->g.ny) return fail(YB_INVALID_ARGUMENT, "peer x/y extents differ");
  if (other->device != s->device) {  // slabs on two GPUs of one process: my kernels store into its memory
    int can = 0;
    YB_CU(cudaDeviceCanAccessPeer(&can, s->device, other->device));
    if (!can)
      return fail(YB_INVALID_ARGUMENT, "device %d cannot access device %d's memory (no P2P path)", s->device,
                  other->device);
    YB_CU(cudaSetDevice(s->device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(other->device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      (void)cudaGetLastError();  // clear the sticky-free "already enabled" status
    else
      YB_CU(e);
  }
  PeerSide& ps = s->peer[side];
  for (int b = 0; b < 2; ++b)
    for (int c = 0; c < 6; ++c) ps.buf[b][c] = other->buf[b][c];
  ps.flags = other->pflags;
  ps.nz = other->g.nz;
  ps.on = true;
  return YB_OK;
}

int yb_peer_push(yb_sim* s, int overlap) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (!s->peer[0].on && !s->peer[1].on) return fail(YB_INVALID_ARGUMENT, "no peer linked");
  YB_CU(cudaSetDevice(s->device));
  const int d = halo_depth(s), nz = s->g.nz;
  const int b = s->pending ? s->cur ^ 1 : s->cur;  // the planes just computed / the current state
  yb::PeerCopy dn{}, up{};
  if (s->peer[0].on) {  // my planes 0..d-1 -> the lower slab's ghosts nz_b..nz_b+d-1
    for (int c = 0; c < 6; ++c) dn.src[c] = s->buf[b][c], dn.dst[c] = s->peer[0].buf[b][c];
    dn.src_k0 = 0, dn.dst_k0 = s->peer[0].nz, dn.nplanes = d;
  }
  if (s->peer[1].on) {  // my planes nz-d..nz-1 -> the upper slab's ghosts -d..-1
    for (int c = 0; c < 6; ++c) up.src[c] = s->buf[b][c], up.dst[c] = s->peer[1].buf[b][c];
    up.src_k0 = nz - d, up.dst_k0 = -d, up.nplanes = d;
  }
  cudaStream_t st = s->stream;
  if (overlap) {  // on a side stream, concurrent with what follows on the main stream
    if (!s->peer_stream) {
      YB_CU(cudaStreamCreateWithFlags(&s->peer_stream, cudaStreamNonBlocking));
      YB_CU(cudaEventCreateWithFlags(&s->peer_go, cudaEventDisableTiming));
      YB_CU(cudaEventCreateWithFlags(&s->peer_done, cudaEventDisableTiming));
    }
    YB_CU(cudaEventRecord(s->peer_go, s->stream));
    YB_CU(cudaStreamWaitEvent(s->peer_stream, s->peer_go, 0));
    st = s->peer_stream;
  }
  YB_CU(yb::launch_peer_copy(s->g, dn, up, st));
  ++s->push_count;
  YB_CU(yb::launch_peer_signal(s->peer[0].on ? s->peer[0].flags + 1 : nullptr,
                               s->peer[1].on ? s->peer[1].flags + 0 : nullptr, s->push_count, st));
  if (overlap) {
    YB_CU(cudaEventRecord(s->peer_done, st));
    s->peer_inflight = true;
  }
  return YB_OK;
}

int yb_peer_step(yb_sim* s, int64_t nsteps) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (!s->peer[0].on && !s->peer[1].on) return fail(YB_INVALID_ARGUMENT, "no peer linked");
  if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight");
  if (nsteps < 1 || nsteps > halo_depth(s)) return fail(YB_INVALID_ARGUMENT, "peer step: 1 .. halo depth steps");
  YB_CU(cudaSetDevice(s->device));
  if (nsteps == 2 && s->variant == YB_VARIANT_TB2) {  // the sweep itself stores the halo (MODE 3)
    if (int rc = prepare_fused(s)) return rc;
    s->q_valid = false;  // this launch does not maintain the quiescent map
    s->peer_stores = true;
    const int rc = step_tb2(s, zfull(s), s->zchunk2, true);
    s->peer_stores = false;
    if (rc) return rc;
    s->step_index += 2;
    s->steps += 2;
    ++s->push_count;
    if (!s->peer_folded)
      YB_CU(yb::launch_peer_signal(s->peer[0].on ? s->peer[0].flags + 1 : nullptr,
                                   s->peer[1].on ? s->peer[1].flags + 0 : nullptr, s->push_count, s->stream));
    s->peer_folded = false;
    return YB_OK;
  }
  if (int rc = yb_peer_wait(s)) return rc;
  if (int rc = yb_advance_begin(s, nsteps)) return rc;  // one step: split sweep + push
  if (int rc = yb_peer_push(s, 0)) return rc;
  return yb_advance_end(s);
}

// Chained exchange periods: nsteps / 2 two-step periods of one slab (a rank:
// n = 1, its neighbours run the same call on their GPUs) or of n linked slabs
// of this device (the one-GPU emulation of n ranks) in ONE persistent launch
// (k_tb2 MODE 4): per sweep, the boundary z-chunks' items wait for the
// neighbours' previous sweep, store their boundary planes into the neighbours'
// ghost planes and signal; the sweeps follow each other through MODE 2's
// device-side neighbourhood counts. Needs the first exchange (yb_peer_push)
// done, like yb_peer_step.
namespace {
constexpr int kChainSweeps = 1024;  // sweeps per launch (longer runs take several launches)

int chain_zchunk(const yb_sim* s) {  // the multi-sweep chunk, with both end chunks >= 2 planes
  const int nz = s->g.nz;
  int len = s->zchunk2p > 0 ? s->zchunk2p : s->zchunk2;
  len = std::max(2, std::min(len, nz));
  while (len < nz && nz % len == 1) ++len;  // a 1-plane top chunk cannot hold the folded exchange
  return len;
}
}  // namespace

int yb_peer_run(yb_sim* const* sims, int n, int64_t nsteps) {
  if (!sims || n < 1 || n > yb::kChainMax) return fail(YB_INVALID_ARGUMENT, "1 .. %d slabs", yb::kChainMax);
  if (nsteps < 2 || (nsteps & 1)) return fail(YB_INVALID_ARGUMENT, "chained periods advance an even step count");
  yb_sim* s0 = sims[0];
  for (int i = 0; i < n; ++i) {
    yb_sim* s = sims[i];
    if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
    // (a handle without peers is a chain of one: plain multi-sweep periods through this path)
    if (s->variant != YB_VARIANT_TB2) return fail(YB_INVALID_ARGUMENT, "chained periods need the two-step kernel");
    if (s->pending) return fail(YB_INVALID_ARGUMENT, "a split sweep is in flight");
    if (!s->probes.empty()) return fail(YB_INVALID_ARGUMENT, "probes sample single steps: use yb_peer_step");
    if (s->device != s0->device || s->g.nx != s0->g.nx || s->g.ny != s0->g.ny || cell_mask(s) != cell_mask(s0))
      return fail(YB_INVALID_ARGUMENT, "slabs of one launch share device, x/y extents and coefficient set");
    if (s->g.nz < 2) return fail(YB_INVALID_ARGUMENT, "slab %d thinner than the two-plane exchange", i);
    for (int j = 0; j < i; ++j)
      if (sims[j] == s) return fail(YB_INVALID_ARGUMENT, "slab %d listed twice", i);
  }
  YB_CU(cudaSetDevice(s0->device));
  if (!s0->chain_ev) YB_CU(cudaEventCreateWithFlags(&s0->chain_ev, cudaEventDisableTiming));
  for (int i = 0; i < n; ++i) {
    yb_sim* s = sims[i];
    if (int rc = prepare_fused(s)) return rc;
    if (!s->pcnt4) YB_CU(cudaMalloc(&s->pcnt4, 2 * kChainSweeps * sizeof(unsigned)));
    if (s->peer_inflight) {  // a push still reading my planes
      YB_CU(cudaStreamWaitEvent(s0->stream, s->peer_done, 0));
      s->peer_inflight = false;
    }
    if (s != s0) {  // everything queued on the other slabs' streams comes first
      if (!s->chain_ev) YB_CU(cudaEventCreateWithFlags(&s->chain_ev, cudaEventDisableTiming));
      YB_CU(cudaEventRecord(s->chain_ev, s->stream));
      YB_CU(cudaStreamWaitEvent(s0->stream, s->chain_ev, 0));
    }
  }
  cudaStream_t st = s0->stream;
  for (int64_t done = 0; done < nsteps;) {
    const int K = (int)std::min<int64_t>((nsteps - done) / 2, kChainSweeps);
    std::vector<yb::ChainSlab> cs(n);
    yb::FusedArgs c{};  // the launch's own arguments: schedule and the chain
    c.nchain = n;
    for (int i = 0; i < n; ++i) {
      yb_sim* s = sims[i];
      const int nxt = s->cur ^ 1;
      yb::FusedArgs& a = cs[i].a;
      a = yb::FusedArgs{};
      a.g = s->g;
      a.nstages = s->stages2;
      a.ntx = s->ntx;
      a.nty = s->nty;
      set_chunks(s, a, chain_zchunk(s), zfull(s));
      a.nsweeps = K;
      a.err = s->werr;
      a.wait_ns = s->wait_ns;
      for (int q = 0; q < 6; ++q) {  // even sweeps write nxt, odd ones cur: the neighbours' same buffers
        a.pdn[q] = s->peer[0].on ? s->peer[0].buf[nxt][q] : nullptr;
        a.pup[q] = s->peer[1].on ? s->peer[1].buf[nxt][q] : nullptr;
        a.pdn_o[q] = s->peer[0].on ? s->peer[0].buf[s->cur][q] : nullptr;
        a.pup_o[q] = s->peer[1].on ? s->peer[1].buf[s->cur][q] : nullptr;
      }
      a.pdn_k0 = s->peer[0].nz;
      a.pfold = 1;
      a.pflag = s->pflags;
      a.pneed = s->push_count;
      a.psig_val = s->push_count + 1;
      a.psig[0] = s->peer[0].on ? s->peer[0].flags + 1 : nullptr;
      a.psig[1] = s->peer[1].on ? s->peer[1].flags + 0 : nullptr;
      a.pcnt = s->pcnt4;
      YB_CU(cudaMemsetAsync(s->pcnt4, 0, 2 * (size_t)K * sizeof(unsigned), st));
      a.perr = s->werr;
      if (s->done_n != a.nitems) {
        cudaFree(s->done);
        s->done = nullptr;
        YB_CU(cudaMalloc(&s->done, (size_t)a.nitems * sizeof(unsigned)));
        YB_CU(cudaMemsetAsync(s->done, 0, (size_t)a.nitems * sizeof(unsigned), st));
        s->done_n = a.nitems;
        s->epoch = 0;
      }
      if (s->srcs_cap < K) {
        cudaFree(s->srcs_dev);
        s->srcs_dev = nullptr;
        YB_CU(cudaMalloc(&s->srcs_dev, (size_t)K * sizeof(yb::SrcArgs)));
        s->srcs_cap = K;
      }
      std::vector<yb::SrcArgs> sv(K);
      for (int q = 0; q < K; ++q) sv[q] = sources_at(s, s->step_index + 2 * q, true);
      YB_CU(cudaMemcpyAsync(s->srcs_dev, sv.data(), sv.size() * sizeof(yb::SrcArgs), cudaMemcpyHostToDevice, st));
      a.done = s->done;
      a.epoch = s->epoch;
      a.srcs = s->srcs_dev;
      a.no_faces = 0;
      a.xblock = s->xblock;
      a.store_policy = 1;
      a.co = coef_args(s);
      for (int q = 0; q < 6; ++q) {
        a.in[q] = s->buf[s->cur][q];
        a.out[q] = s->buf[nxt][q];
      }
      a.src = sources_at(s, s->step_index, true);
      a.skipped = s->qskipped;
      cs[i].tm = s->tm2[s->cur];
      cs[i].tm_o = s->tm2[nxt];
      c.chain_off[i + 1] = c.chain_off[i] + a.nitems;
    }
    c.g = s0->g;
    c.nstages = s0->stages2;
    c.pf = s0->pf2;
    c.ntx = s0->ntx;
    c.nty = s0->nty;
    c.xblock = s0->xblock;
    c.nsweeps = K;
    c.nitems = c.chain_off[n];
    c.sched = s0->sched;
    c.sched_base = s0->sched_base;
    c.err = s0->werr;
    c.wait_ns = s0->wait_ns;
    const int mask = cell_mask(s0);
    const size_t smem = yb::tb2_smem_bytes(mask, s0->stages2);
    const dim3 grid(std::min(c.nitems, s0->num_sms), 1, 1);
    TimerPair* tp = nullptr;
    if (s0->timing) {
      if (s0->timers_used == s0->timers.size()) {
        TimerPair p;
        YB_CU(cudaEventCreate(&p.a));
        YB_CU(cudaEventCreate(&p.b));
        s0->timers.push_back(p);
      }
      tp = &s0->timers[s0->timers_used++];
      YB_CU(cudaEventRecord(tp->a, st));
    }
    if (n == 1) {  // a rank's launch: the slab's own arguments as the kernel's, maps as parameters
      yb::FusedArgs a1 = cs[0].a;
      a1.nchain = 1;
      a1.chain_off[0] = 0;
      a1.chain_off[1] = a1.nitems;
      a1.nsweeps = K;
      a1.sched = c.sched;
      a1.sched_base = c.sched_base;
      a1.pf = c.pf;
      YB_CU(yb::launch_tb2(a1, cs[0].tm, cs[0].tm_o, mask, grid, smem, st));
    } else {
      YB_CU(yb::launch_tb2_chain(c, cs.data(), n, mask, grid, smem, st));
    }
    if (tp) YB_CU(cudaEventRecord(tp->b, st));
    s0->sched_base += (unsigned long long)c.nitems * K + grid.x;
    s0->launches += 1;
    for (int i = 0; i < n; ++i) {
      yb_sim* s = sims[i];
      s->epoch += (unsigned)K;
      s->push_count += (unsigned)K;
      s->step_index += 2 * K;
      s->steps += 2 * K;
      if (K & 1) s->cur ^= 1;
      s->q_valid = false;  // MODE 4 does not maintain the quiescent map
    }
    done += 2 * K;
  }
  YB_CU(cudaEventRecord(s0->chain_ev, st));
  for (int i = 1; i < n; ++i) YB_CU(cudaStreamWaitEvent(sims[i]->stream, s0->chain_ev, 0));
  return YB_OK;
}

int yb_peer_wait(yb_sim* s) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (!s->pflags) return fail(YB_INVALID_ARGUMENT, "no peer linked");
  YB_CU(cudaSetDevice(s->device));
  if (s->peer_inflight) {  // my own push must have read my planes before they are rewritten
    YB_CU(cudaStreamWaitEvent(s->stream, s->peer_done, 0));
    s->peer_inflight = false;
  }
  YB_CU(yb::launch_peer_wait(s->pflags, s->peer[0].on ? s->push_count : 0u, s->peer[1].on ? s->push_count : 0u,
                             s->werr, s->wait_ns, s->stream));
  if (s->qskip && s->q_valid) {  // the neighbours stored my ghost planes: mark their nonzero tile-planes
    const int d = halo_depth(s);  // (yb_halo_unpack does the same for the NCCL transport)
    if (s->peer[0].on)
      YB_CU(yb::launch_qscan(s->g, fields_of(s, 0), fields_of(s, 1), qmap_of(s), -d, -1, s->stream));
    if (s->peer[1].on)
      YB_CU(yb::launch_qscan(s->g, fields_of(s, 0), fields_of(s, 1), qmap_of(s), s->g.nz, s->g.nz + d - 1,
                             s->stream));
  }
  return YB_OK;
}

int yb_set_quiescent_skip(yb_sim* s, int on) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  s->qskip = on != 0;
  s->q_valid = false;
  return YB_OK;
}

int yb_set_stream(yb_sim* s, void* stream) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  YB_CU(cudaSetDevice(s->device));
  YB_CU(cudaStreamSynchronize(s->stream));
  s->stream = stream ? static_cast<cudaStream_t>(stream) : s->own_stream;
  return YB_OK;
}

int yb_set_kernel_timing(yb_sim* s, int on) {
  if (!s) return fail(YB_INVALID_ARGUMENT, "null handle");
  if (int rc = collect_timers(s)) return rc;
  s->timing = on != 0;
  s->kernel_ms = 0.0;
  s->kernel_timed = 0;
  return YB_OK;
}

int yb_get_info(yb_sim* s, yb_info* info) {
  if (!s || !info) return fail(YB_INVALID_ARGUMENT, "null argument");
  YB_CU(cudaSetDevice(s->device));
  if (int rc = collect_timers(s)) return rc;
  if (s->variant != YB_VARIANT_NAIVE)
    if (int rc = prepare_fused(s)) return rc;
  std::memset(info, 0, sizeof *info);
  info->step_index = s->step_index;
  info->steps = s->steps;
  info->kernel_launches = s->launches;
  info->main_kernel_ms = s->kernel_ms;
  info->main_kernel_timed = s->kernel_timed;
  info->n_cell_arrays = popcount4(cell_mask(s));
  info->variant = s->variant;
  info->stages = s->stages;
  info->grid_x = (int)s->grid.x;
  info->grid_y = (int)s->grid.y;
  info->grid_z = (int)s->grid.z;
  info->zchunk = s->zchunk;
  info->bytes_per_cell_update = (48.0 + 4.0 * info->n_cell_arrays) /
                                (s->variant == YB_VARIANT_TB2 ? 2.0 : (s->variant == YB_VARIANT_TB4 ? 4.0 : 1.0));
  if (s->variant == YB_VARIANT_TB4) {
    info->stages = s->stages4;
    info->grid_x = std::min(s->ntx4 * s->nty4 * ((s->g.nz + s->zchunk4 - 1) / s->zchunk4), s->num_sms);
    info->zchunk = s->zchunk4;
  } else if (s->variant == YB_VARIANT_TB2) {
    info->stages = s->stages2;
    info->grid_x = (int)s->grid2.x;
    info->zchunk = (s->persist && s->zchunk2p > 0 && s->g.nzg == s->g.nz && !s->qskip) ? s->zchunk2p : s->zchunk2;
  }
  info->device_bytes = s->dev_bytes;
  info->halo_depth = halo_depth(s);
  info->quiescent_skip = s->qskip ? 1 : 0;
  if (s->qskipped) {
    unsigned long long v = 0;
    YB_CU(cudaMemcpyAsync(&v, s->qskipped, sizeof v, cudaMemcpyDeviceToHost, s->stream));
    YB_CU(cudaStreamSynchronize(s->stream));
    info->skipped_items = (int64_t)v;
  }
  info->streamed_readbacks = s->streamed;
  info->streamed_uploads = s->streamed_up;
  return YB_OK;
}

}  // extern "C"

// ------------------------------------------- per-box ops on host FieldSets
namespace {

struct IBox {
  int lo[3], hi[3];
  bool empty() const { return hi[0] <= lo[0] || hi[1] <= lo[1] || hi[2] <= lo[2]; }
};

IBox ibox(const int* b) { return {{b[0], b[2], b[4]}, {b[1], b[3], b[5]}}; }

// contains (array3.hpp:47-52): an empty inner box is contained in anything
bool box_contains(const IBox& outer, const IBox& inner) {
  if (inner.empty()) return true;
  for (int a = 0; a < 3; ++a)
    if (inner.lo[a] < outer.lo[a] || inner.hi[a] > outer.hi[a]) return false;
  return true;
}

IBox box_intersect(const IBox& p, const IBox& q) {
  IBox r;
  for (int a = 0; a < 3; ++a) {
    r.lo[a] = std::max(p.lo[a], q.lo[a]);
    r.hi[a] = std::min(p.hi[a], q.hi[a]);
  }
  return r;
}

// comp_extents / curl_updatable_box (staggering.hpp:59-77)
IBox extents_box(const int n[3], int c) {
  IBox b;
  const int axis = c % 3;
  for (int a = 0; a < 3; ++a) {
    const bool node = c < 3 ? (a != axis) : (a == axis);
    b.lo[a] = 0;
    b.hi[a] = n[a] + (node ? 1 : 0);
  }
  return b;
}

IBox updatable_box(const int n[3], int c) {
  IBox b = extents_box(n, c);
  if (c < 3)
    for (int a = 0; a < 3; ++a)
      if (a != c % 3) b.lo[a] = 1, b.hi[a] = n[a];
  return b;
}

struct SubOp {
  int op, comp;
  IBox box;
};

// The component-boxes an operation updates, with the reference's range checks.
int plan_fs_op(const int n[3], int op, int comp, const int* box, std::vector<SubOp>& out) {
  const IBox node = {{0, 0, 0}, {n[0] + 1, n[1] + 1, n[2] + 1}};  // detail::node_box, kernels.hpp:113-116
  switch (op) {
    case YB_OP_UPDATE_E: {  // update_e_box, kernels.hpp:78-88
      if (comp < 0 || comp > 2) return fail(YB_INVALID_ARGUMENT, "update_e_box: component %d is not electric", comp);
      const IBox b = ibox(box);
      if (b.empty()) return YB_OK;
      if (!box_contains(updatable_box(n, comp), b))
        return fail(YB_OUT_OF_RANGE, "update_e_box: box outside updatable range");
      out.push_back({0, comp, b});
      return YB_OK;
    }
    case YB_OP_UPDATE_H: {  // update_h_box, kernels.hpp:92-101
      if (comp < 3 || comp > 5) return fail(YB_INVALID_ARGUMENT, "update_h_box: component %d is not magnetic", comp);
      const IBox b = ibox(box);
      if (b.empty()) return YB_OK;
      if (!box_contains(extents_box(n, comp), b))
        return fail(YB_OUT_OF_RANGE, "update_h_box: box outside component extents");
      out.push_back({1, comp, b});
      return YB_OK;
    }
    case YB_OP_ZERO: {  // zero_box, kernels.hpp:104-111
      if (comp < 0 || comp > 5) return fail(YB_INVALID_ARGUMENT, "zero_box: component %d", comp);
      const IBox b = ibox(box);
      if (b.empty()) return YB_OK;
      if (!box_contains(extents_box(n, comp), b))
        return fail(YB_OUT_OF_RANGE, "zero_box: box outside component extents");
      out.push_back({2, comp, b});
      return YB_OK;
    }
    case YB_OP_AMPERE:
    case YB_OP_FARADAY: {  // apply_ampere_range / apply_faraday_range, kernels.hpp:129-144
      const IBox b = ibox(box);
      const bool amp = op == YB_OP_AMPERE;
      if (!box_contains(node, b))  // detail::check_range, kernels.hpp:118-122
        return fail(YB_OUT_OF_RANGE, "%s: range out of bounds", amp ? "apply_ampere_range" : "apply_faraday_range");
      for (int c = amp ? 0 : 3; c < (amp ? 3 : 6); ++c) {
        const IBox r = box_intersect(b, amp ? updatable_box(n, c) : extents_box(n, c));
        if (!r.empty()) out.push_back({amp ? 0 : 1, c, r});
      }
      return YB_OK;
    }
    case YB_OP_PEC:  // apply_pec_boundary, kernels.hpp:147-155: the tangential node planes of each face
      for (int c = 0; c < 3; ++c) {
        const IBox ext = extents_box(n, c);
        for (int a = 0; a < 3; ++a) {
          if (a == c) continue;
          for (int side = 0; side < 2; ++side) {
            IBox r = ext;
            r.lo[a] = side ? n[a] : 0;
            r.hi[a] = r.lo[a] + 1;
            out.push_back({2, c, r});
          }
        }
      }
      return YB_OK;
    default:
      return fail(YB_INVALID_ARGUMENT, "unknown operation %d", op);
  }
}

// components an update of `comp` reads (kernels.hpp:18-25)
int stencil_mask(int op, int comp) {
  if (op == 2) return 1 << comp;
  static const int reads[6] = {(1 << 5) | (1 << 4), (1 << 3) | (1 << 5), (1 << 4) | (1 << 3),
                               (1 << 1) | (1 << 2), (1 << 2) | (1 << 0), (1 << 0) | (1 << 1)};
  return (1 << comp) | reads[comp];
}

template <class T>
int fs_apply_t(int device, const int n[3], void* const* dense6, const void* const* cd3,
               const std::vector<SubOp>& ops) {
  yb::HostExt x{};
  for (int c = 0; c < 6; ++c) {
    const IBox e = extents_box(n, c);
    for (int a = 0; a < 3; ++a) x.e[c][a] = e.hi[a];
  }
  int rd = 0, wr = 0;
  bool need_cd = false;
  for (const SubOp& o : ops) {
    rd |= stencil_mask(o.op, o.comp);
    wr |= 1 << o.comp;
    need_cd |= o.op != 2;
  }
  for (int c = 0; c < 6; ++c)
    if (((rd | wr) >> c & 1) && !dense6[c]) return fail(YB_INVALID_ARGUMENT, "component %d array is null", c);
  if (need_cd && (!cd3 || !cd3[0] || !cd3[1] || !cd3[2]))
    return fail(YB_INVALID_ARGUMENT, "coefficient arrays are null");
  YB_CU(cudaSetDevice(device));
  yb::HostFields<T> f{};
  void* mem[9] = {};
  auto release = [&](int rc) {
    for (void* p : mem) cudaFree(p);
    return rc;
  };
  for (int c = 0; c < 6; ++c) {
    if (!((rd | wr) >> c & 1)) continue;
    const size_t bytes = (size_t)x.e[c][0] * x.e[c][1] * x.e[c][2] * sizeof(T);
    if (cudaMalloc(&mem[c], bytes) != cudaSuccess ||
        yb::copy_h2d(mem[c], dense6[c], bytes, 0) != cudaSuccess)
      return release(fail(YB_CUDA_ERROR, "host FieldSet: copy of component %d to the device failed", c));
    f.f[c] = static_cast<T*>(mem[c]);
  }
  if (need_cd)
    for (int a = 0; a < 3; ++a) {
      const size_t bytes = (size_t)n[a] * sizeof(T);
      if (cudaMalloc(&mem[6 + a], bytes) != cudaSuccess ||
          cudaMemcpy(mem[6 + a], cd3[a], bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        return release(fail(YB_CUDA_ERROR, "coefficient copy failed"));
      f.cd[a] = static_cast<const T*>(mem[6 + a]);
    }
  // in the reference's order: components one after another (stream-ordered)
  for (const SubOp& o : ops) {
    const yb::HostBox b{o.box.lo[0], o.box.hi[0], o.box.lo[1], o.box.hi[1], o.box.lo[2], o.box.hi[2]};
    if (yb::launch_host_box<T>(f, x, o.op, o.comp, b, 0) != cudaSuccess)
      return release(fail(YB_CUDA_ERROR, "per-box kernel launch failed"));
  }
  for (int c = 0; c < 6; ++c) {
    if (!(wr >> c & 1)) continue;
    const size_t bytes = (size_t)x.e[c][0] * x.e[c][1] * x.e[c][2] * sizeof(T);
    if (yb::copy_d2h(dense6[c], mem[c], bytes, 0) != cudaSuccess)
      return release(fail(YB_CUDA_ERROR, "host FieldSet: copy of component %d back failed", c));
  }
  if (cudaStreamSynchronize(0) != cudaSuccess) return release(fail(YB_CUDA_ERROR, "host FieldSet: copy back failed"));
  return release(YB_OK);
}

template <class T>
int fs_energy_t(int device, const int n[3], const void* const* dense6, const void* const* prev3,
                const double* const* d3, double* energy) {
  yb::HostExt x{};
  for (int c = 0; c < 6; ++c) {
    const IBox e = extents_box(n, c);
    for (int a = 0; a < 3; ++a) x.e[c][a] = e.hi[a];
  }
  YB_CU(cudaSetDevice(device));
  void* mem[10] = {};
  auto release = [&](int rc) {
    for (void* p : mem) cudaFree(p);
    return rc;
  };
  yb::HostFields<T> f{};
  const T* prev[3] = {};
  for (int q = 0; q < 9; ++q) {
    const int c = q < 6 ? q : q - 3;
    const size_t bytes = (size_t)x.e[c][0] * x.e[c][1] * x.e[c][2] * sizeof(T);
    const void* src = q < 6 ? dense6[q] : prev3[q - 6];
    if (cudaMalloc(&mem[q], bytes) != cudaSuccess || cudaMemcpy(mem[q], src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      return release(fail(YB_CUDA_ERROR, "total_energy: copy to the device failed"));
    if (q < 6)
      f.f[q] = static_cast<T*>(mem[q]);
    else
      prev[q - 6] = static_cast<const T*>(mem[q]);
  }
  std::vector<double> dxyz;
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n[a]; ++i) dxyz.push_back(d3[a] ? d3[a][i] : 1.0);
  const size_t scratch = (size_t)yb::host_energy_scratch_doubles();
  if (cudaMalloc(&mem[9], (dxyz.size() + scratch) * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(mem[9], dxyz.data(), dxyz.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return release(fail(YB_CUDA_ERROR, "total_energy: spacing copy failed"));
  double* d = static_cast<double*>(mem[9]);
  if (yb::launch_host_energy<T>(f, prev, x, d, n[0], n[1], n[2], d + dxyz.size(), 0) != cudaSuccess ||
      cudaMemcpy(energy, d + dxyz.size() + scratch - 1, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return release(fail(YB_CUDA_ERROR, "total_energy kernel failed"));
  return release(YB_OK);
}

}  // namespace

extern "C" {

int yb_fs_apply(int device, int dtype, int nx, int ny, int nz, void* const* dense6, const void* const* cd3, int op,
                int comp, const int* box) {
  if (!dense6) return fail(YB_INVALID_ARGUMENT, "null field arrays");
  if (dtype != YB_F32 && dtype != YB_F64) return fail(YB_INVALID_ARGUMENT, "unknown element type %d", dtype);
  if (nx < 1 || ny < 1 || nz < 1) return fail(YB_INVALID_ARGUMENT, "cell counts must be positive");
  if (op != YB_OP_PEC && !box) return fail(YB_INVALID_ARGUMENT, "null box");
  const int n[3] = {nx, ny, nz};
  std::vector<SubOp> ops;
  if (int rc = plan_fs_op(n, op, comp, box, ops)) return rc;
  if (ops.empty()) return YB_OK;
  return dtype == YB_F32 ? fs_apply_t<float>(device, n, dense6, cd3, ops)
                         : fs_apply_t<double>(device, n, dense6, cd3, ops);
}

int yb_fs_total_energy(int device, int dtype, int nx, int ny, int nz, const void* const* dense6,
                       const void* const* prev_h3, const double* dx, const double* dy, const double* dz,
                       double* energy) {
  if (!dense6 || !prev_h3 || !energy) return fail(YB_INVALID_ARGUMENT, "null argument");
  for (int c = 0; c < 6; ++c)
    if (!dense6[c] || (c < 3 && !prev_h3[c])) return fail(YB_INVALID_ARGUMENT, "null array");
  if (dtype != YB_F32 && dtype != YB_F64) return fail(YB_INVALID_ARGUMENT, "unknown element type %d", dtype);
  if (nx < 1 || ny < 1 || nz < 1) return fail(YB_INVALID_ARGUMENT, "cell counts must be positive");
  const int n[3] = {nx, ny, nz};
  const double* d3[3] = {dx, dy, dz};
  return dtype == YB_F32 ? fs_energy_t<float>(device, n, dense6, prev_h3, d3, energy)
                         : fs_energy_t<double>(device, n, dense6, prev_h3, d3, energy);
}

}  // extern "C"
