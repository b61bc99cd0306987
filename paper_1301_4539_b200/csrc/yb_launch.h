// yb_launch.h — host-side launch wrappers shared between the kernel TUs and
// the C-ABI implementation (yb_capi.cu). Internal; not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <mutex>

#include "yb_device.cuh"

namespace yb {

// Fused sweep geometry (yb_fused.cu).
constexpr int kTX = 128;            // owned cells along x per CTA (32 lanes x float4)
constexpr int kTY = 8;              // owned rows per CTA = consumer warps; warp kTY = TMA producer
constexpr int kWarps = kTY + 2;    // + producer warp + face warp
constexpr int kThreads = 32 * kWarps;
constexpr int kBX = kTX + 8;        // staged box: x0-4 .. x0+TX+3 (16-byte TMA rows)
constexpr int kBY = kTY + 2;        // staged box: y0-1 .. y0+TY
constexpr int kSlot = ((kBX * kBY * 4 + 127) / 128) * 32;  // floats per array slot (128-B aligned)
constexpr int kMaxArrays = 10;      // 6 fields + up to 4 per-cell coefficient arrays

// Two-step (temporal depth 2) sweep geometry (yb_tb2.cu): 8 output rows,
// staged rows y0-2..y0+9, row warps for rows y0-1..y0+9, one edge-column
// warp, one TMA producer warp, one face warp.
constexpr int kTB2Rows = 8;
constexpr int kTB2BY = kTB2Rows + 4;                  // staged box rows
constexpr int kTB2RowWarps = kTB2Rows + 3;            // E1 rows
constexpr int kTB2Warps = kTB2RowWarps + 3;           // + edge, producer, face
constexpr int kTB2Threads = 32 * kTB2Warps;
// Staged rows per array: fields y0-2..y0+9 (12), Ca/Cb y0-1..y0+9 (11),
// Da/Db y0-1..y0+8 (10) — each array only as tall as its consumers need.
constexpr int kTB2RowsCA = kTB2Rows + 3;
constexpr int kTB2RowsDA = kTB2Rows + 2;
constexpr int slot_floats(int rows) { return ((kBX * rows * 4 + 127) / 128) * 32; }
constexpr int kTB2SlotF = slot_floats(kTB2BY);
// ex, ey, ez, hy are read on rows y0-1 .. y0+9 only (hx, hz also on y0-2,
// for the j-1 neighbour of row y0-1): 11-row boxes for those four, which
// trims a stage enough for a third one next to a per-cell Cb array.
constexpr int kTB2RowsE = kTB2Rows + 3;
constexpr int kTB2SlotE = slot_floats(kTB2RowsE);
__host__ __device__ constexpr bool tb2_short(int q) { return q != 3 && q != 5; }  // ex, ey, ez, hy
// physical start (floats) of component q's slot in a stage: ex, ey, ez, hx, hy, hz
__host__ __device__ constexpr int tb2_foff(int q) {
  return q <= 3 ? q * kTB2SlotE : (q == 4 ? 3 * kTB2SlotE + kTB2SlotF : 4 * kTB2SlotE + kTB2SlotF);
}
// the slot's row-y0-2 origin (the 11-row slots start one row lower)
__host__ __device__ constexpr int tb2_fbase(int q) { return tb2_foff(q) - (tb2_short(q) ? kBX : 0); }
constexpr int kTB2Fields = 4 * kTB2SlotE + 2 * kTB2SlotF;  // floats of the six field slots
constexpr int kTB2SlotC = slot_floats(kTB2RowsCA);
constexpr int kTB2SlotD = slot_floats(kTB2RowsDA);
constexpr int kTB2E1 = 2 * 3 * kTB2RowWarps * kBX;    // E^{n+1} planes (double buffered)
constexpr int kTB2H1 = 2 * 3 * (kTB2Rows + 2) * kBX;  // H^{n+3/2} planes (double buffered)
constexpr int kTB2E2 = 2 * 3 * (kTB2Rows + 1) * kBX;  // E^{n+2} planes (double buffered)
constexpr int kTB2Edge = 2 * 3 * kTB2RowWarps * 3 + 2 * 2 * (kTB2Rows + 2) * 2 + 2 * 2 * kTB2RowWarps;

// Four-step (temporal depth 4) sweep geometry (yb_tb4.cu): 4 output rows x
// 56 output columns; every warp works on an 11-row x 64-column window.
constexpr int kTB4Rows = 4;
constexpr int kTB4RowWarps = kTB4Rows + 7;  // window rows y0-3 .. y0+7
constexpr int kTB4BY = kTB4RowWarps + 1;    // staged field rows y0-4 .. y0+7
constexpr int kTB4Win = 64;                 // window columns x0-4 .. x0+59
constexpr int kTB4Cols = kTB4Win - 8;       // output columns x0 .. x0+55

// floats of one stage for a coefficient set (mask bit q: array q per-cell)
inline int tb2_stage_floats(int cell_mask) {
  return kTB2Fields + ((cell_mask & 1) + ((cell_mask >> 1) & 1)) * kTB2SlotC +
         (((cell_mask >> 2) & 1) + ((cell_mask >> 3) & 1)) * kTB2SlotD;
}

inline size_t tb2_smem_bytes(int cell_mask, int stages) {
  return (size_t)stages * tb2_stage_floats(cell_mask) * 4 + (size_t)(kTB2E1 + kTB2H1 + kTB2E2 + kTB2Edge) * 4 +
         (size_t)stages * 16 + 24 * 4;  // mbarriers, item + sweep + slab queues
}

struct TMaps {
  CUtensorMap m[kMaxArrays];  // read side: ex..hz of the current state, then cell coeffs
};

struct FusedArgs {
  Geo g;
  int nstages;
  int pf;  // two-step producer: L2 prefetch (cp.async.bulk.prefetch.tensor) this many planes ahead (0: off)
  int zchunk;
  // z-chunks of this launch: nch0 chunks over planes [zb0, ze0), then the
  // rest over [zb1, ze1) (a whole sweep: [0, nz) and an empty second range;
  // split sweeps: the slab's boundary planes, or its interior)
  int zb0, ze0, zb1, ze1, nch0;
  int ntx, nty;  // tiles along x, y
  int nitems;    // work items = tiles * z-chunks, handed out by *sched
  unsigned long long* sched;     // monotonic global work counter
  unsigned long long sched_base; // counter value at this launch's start
  int store_policy;              // L2 policy of next-state stores: 0 normal, 1 evict_first, 2 unchanged
  CoefArgs co;
  const float* in[6];
  float* out[6];
  SrcArgs src;
  QMap qm;                       // quiescent map (qm.bits == nullptr: off)
  unsigned long long* skipped;   // skipped-item counter
  // Several sweeps in one launch (two-step kernel, single domain): sweep s
  // reads in[] for even s / out[] for odd s and writes the other; an item of
  // sweep s >= 1 starts once its neighbourhood finished sweep s-1
  // (done[item] >= epoch + s), and publishes done[item] = epoch + s + 1.
  int nsweeps;                   // 1: an ordinary launch
  unsigned* done;                // per-item completion epochs
  unsigned epoch;
  const SrcArgs* srcs;           // per-sweep sources (nsweeps > 1)
  int* err;                      // wait-error record (WaitErr) of a timed-out dependency wait
  unsigned long long wait_ns;    // deadline of every spin wait of this launch (ns of globaltimer)
  // Peer-store mode (two-step kernel MODE 3, z-slabs over peer memory): the
  // boundary planes 0,1 / nz-2,nz-1 this launch writes also go straight into
  // the neighbours' ghost planes pdn_k0 + {0,1} / {-2,-1} of the same-parity
  // buffers (NVLink stores, overlapped with the rest of the sweep).
  float* pdn[6];                 // slab below (nullptr: none)
  float* pup[6];                 // slab above
  int pdn_k0;                    // the lower slab's depth (its ghost plane for my plane 0)
  // ... with the exchange's ordering folded in (pfold): the bottom / top z-chunk's
  // items run first, each waits (bounded) for my flag word pflag[0] / pflag[1] >=
  // pneed before loading the ghost planes that neighbour writes (and before writing
  // its), and the last of them to finish publishes psig_val to that neighbour's flag
  // word psig[0] / psig[1] — no wait or signal launches, and a neighbour can start
  // its next period's boundary items while this launch is still in its interior.
  int pfold;
  const unsigned* pflag;
  // the upper-face DoFs are someone else's: the interior launch of a split
  // sweep runs concurrently with the boundary launch, which applies them
  // (the two-step update h <- f(f(h)) re-reads its output, so it must run once)
  int no_faces;
  unsigned pneed, psig_val;
  unsigned* psig[2];
  unsigned* pcnt;                // per side: boundary items completed (monotonic)
  unsigned pcnt_base[2];         // their values at this launch's start
  int* perr;                     // wait-error record of a timed-out neighbour wait
  // Chained exchange periods (two-step kernel MODE 4): nsweeps periods of one
  // or several linked slabs in ONE persistent launch — MODE 2's device-side
  // sweep dependencies plus MODE 3's folded peer stores / waits / signals per
  // sweep. Sweep s stores its boundary planes into the neighbour's buffers of
  // s's output parity (pdn/pup for even s, pdn_o/pup_o for odd s), its
  // boundary items wait for the neighbour's flag >= pneed + s, and the last
  // of a side's row warps of sweep s (counter pcnt[side * nsweeps + s], zeroed
  // per launch) publishes psig_val + s. The launch's own arguments carry
  // nchain slabs (their arguments and read maps are kernel parameters next to
  // these: ChainParams, yb_tb2.cu) and chain_off (items of slabs 0..k-1 per
  // sweep); work item v = (sweep, slab, item). nchain > 1 runs several slabs of
  // one GPU in one launch — the one-GPU emulation of the multi-GPU schedule; a
  // rank runs nchain = 1.
  float* pdn_o[6];
  float* pup_o[6];
  int nchain;
  int chain_off[9];
  // Streamed readback (yb_run_to_host, MODE 2): sweeps skew0.. are handed out
  // along y-skewed diagonals d = 2*(sweep - skew0) + tile_row (diag[d] = (sweep,
  // tile row) groups before diagonal d, ndiag diagonals; the sweeps before
  // skew0 sweep-major) so a tile row finishes its last sweep early; every row warp of a last-sweep item adds 1 to band[tile row]
  // and every face warp to band[nty] (system-scope fence first), so copy-engine
  // readbacks waiting on those counters (cuStreamWaitValue32) overlap the
  // sweeps still running. band == nullptr: sweep-major order, no counting.
  const int* diag;
  int ndiag, skew0;
  unsigned* band;
  // Streamed upload (yb_run_streamed, MODE 2): the mirror image at the launch's
  // start — the first skewh sweeps (skewh <= skew0; their own table diagh / ndiagh)
  // run along the mirrored diagonals, so tile row 0 starts first and the others
  // follow in ascending order, half a sweep apart; a sweep-0 item of tile row
  // ty loads only after upband[min(ty + 1, nty - 1)] >= up_need (the copy
  // stream writes upband[q] = up_need once the host->device copies of tile
  // rows 0..q have landed: cuStreamWriteValue32), and the face warps wait for
  // the last row's word. upband == nullptr: the state is resident.
  int skewh;
  const int* diagh;
  int ndiagh;
  const unsigned* upband;
  unsigned up_need;
  // Multi-sweep launches hand out a sweep's tiles in columns xblock tiles wide (within a z-chunk:
  // column block, then tile row, then tile column), not row by row. Persistent CTAs take items at
  // a steady rate (one every item_time / CTAs: ~1.7 planes of progress on config 4), so two items
  // q queue positions apart run ~1.7 q planes apart, and L2 keeps the rows they share for only
  // ~6-9 planes: row-major order puts y-neighbours ntx (8) positions apart (measured median 11.7
  // planes, tools/stamp_drift.py), a 2-wide column 2. 0 or >= ntx: row-major.
  int xblock;
#ifdef YB_TB2_STAMP  // measurement builds: globaltimer at each item's first and last load (tools/stamp_drift.py)
  unsigned long long* stamp;
#endif
};

constexpr int kChainMax = 8;
struct ChainSlab {
  FusedArgs a;
  TMaps tm, tm_o;  // read maps of the launch's even / odd sweeps
};

// Wait-error record, 8 ints per handle: [0] code (0 none; WAIT_DEP: a
// multi-sweep item waited for its neighbourhood; WAIT_PEER_KERNEL: the
// folded peer wait of a boundary item; WAIT_PEER: the separate peer-wait
// launch; WAIT_UPLOAD: a first-sweep item waited for its tile rows' upload), [1] item (-1 if none), [2] sweep / side, [3] counter value seen,
// [4] value needed.
enum { WAIT_DEP = 1, WAIT_PEER_KERNEL = 2, WAIT_PEER = 3, WAIT_UPLOAD = 4 };

// Position q of a sweep's sweep-major order -> item (FusedArgs::xblock): z-chunk, then column
// block of xblock tiles, then tile row, then tile column within the block (T = tiles per chunk).
__device__ __forceinline__ int block_order(const FusedArgs& a, int q, int T) {
  const int W = a.xblock;
  if (W <= 0 || W >= a.ntx) return q;
  const int ch = q / T, r = q - ch * T;
  const int per = W * a.nty;                   // items of a full column block
  const int b = min(r / per, (a.ntx - 1) / W);  // the last block may be narrower
  const int r2 = r - b * per, wb = min(W, a.ntx - b * W);
  const int ty = r2 / wb, tx = b * W + (r2 - ty * wb);
  return ch * T + ty * a.ntx + tx;
}

// planes [kz0, kz1) of z-chunk c of a launch
__device__ __forceinline__ void chunk_planes(const FusedArgs& a, int c, int& kz0, int& kz1) {
  if (c < a.nch0) {
    kz0 = a.zb0 + c * a.zchunk;
    kz1 = min(kz0 + a.zchunk, a.ze0);
  } else {
    kz0 = a.zb1 + (c - a.nch0) * a.zchunk;
    kz1 = min(kz0 + a.zchunk, a.ze1);
  }
}

// Soft sources of the four steps of one depth-4 launch (bit s of act: the
// source injects at step n+s with increment val[s]).
struct SrcArgs4 {
  int n;
  int comp[kMaxSources], i[kMaxSources], j[kMaxSources], k[kMaxSources];
  float val[kMaxSources][4];
  int act[kMaxSources];
};
size_t tb4_smem_bytes(int cell_mask, int stages);
cudaError_t tb4_set_smem_limits();
cudaError_t launch_tb4(const FusedArgs& a, const SrcArgs4& s, const TMaps& tm, int cell_mask, dim3 grid,
                       size_t smem, cudaStream_t st);

// smem bytes of the fused kernel for `narr` staged arrays and `stages` ring depth.
inline size_t fused_smem_bytes(int narr, int stages) {
  return (size_t)stages * narr * kSlot * 4 + (size_t)stages * 16 + 8 * 4;
}

// cell_mask bit q set <=> coefficient array q (Ca,Cb,Da,Db) is per-cell.
cudaError_t launch_fused(const FusedArgs& a, const TMaps& tm, int cell_mask, dim3 grid,
                         size_t smem, cudaStream_t st);
cudaError_t fused_set_smem_limits();
// Two full steps per launch (maps with kTB2BY-row boxes).
// MODE 4: a = the launch's schedule (nsweeps, nchain, chain_off, sched, ...),
// slabs[0..n) every slab's own arguments and read maps.
cudaError_t launch_tb2_chain(const FusedArgs& a, const ChainSlab* slabs, int n, int cell_mask, dim3 grid,
                             size_t smem, cudaStream_t st);
cudaError_t launch_tb2(const FusedArgs& a, const TMaps& tm, const TMaps& tm_out, int cell_mask, dim3 grid,
                       size_t smem, cudaStream_t st);
cudaError_t tb2_set_smem_limits();

cudaError_t launch_naive_ampere(const Geo& g, const Fields& F, const CoefArgs& co, const int* box,
                                cudaStream_t st);
cudaError_t launch_naive_faraday(const Geo& g, const Fields& F, const CoefArgs& co, const int* box,
                                 cudaStream_t st);
cudaError_t launch_naive_pec(const Geo& g, const Fields& F, cudaStream_t st);
cudaError_t launch_sources(const Geo& g, const Fields& F, const SrcArgs& s, cudaStream_t st);
cudaError_t launch_faces(const Geo& g, const Fields& in, const Fields& out, const CoefArgs& co,
                         int num_sms, cudaStream_t st);
cudaError_t launch_fill_fields(const Geo& g, const Fields& F, uint64_t seed, cudaStream_t st);
cudaError_t launch_medium(const Geo& g, float* ca, float* cb, float* da, float* db,
                          long long eps_seed, long long sigma_seed, float S, cudaStream_t st);
cudaError_t launch_clamp_fill(const Geo& g, float* a, int kmin, int kmax, cudaStream_t st);
cudaError_t launch_scatter_dense(const Geo& g, const int* e, const float* dense, float* padded,
                                 cudaStream_t st);
cudaError_t launch_gather_dense(const Geo& g, const int* e, const float* padded, float* dense,
                                cudaStream_t st);
struct ProbeArgs {
  int n;
  int comp[64];
  long long off[64];
};
// Sets the quiescent bit of every (tile, plane k in [k0, k1]) holding a
// nonzero DoF in either state buffer.
cudaError_t launch_qscan(const Geo& g, const Fields& a, const Fields& b, const QMap& q, int k0, int k1,
                         cudaStream_t st);
// Direct halo push over peer memory (NVLink / same device): copy `nplanes`
// planes of all six components from src (my state) to dst (the neighbour's
// state), then — in a separate launch — publish `epoch` in its flag word.
struct PeerCopy {
  const float* src[6];
  float* dst[6];
  int src_k0, dst_k0, nplanes;  // 0 planes: direction unused
};
cudaError_t launch_peer_copy(const Geo& g, const PeerCopy& down, const PeerCopy& up, cudaStream_t st);
cudaError_t launch_peer_signal(unsigned* flag_down, unsigned* flag_up, unsigned epoch, cudaStream_t st);
// Spins until flags[0] >= need0 and flags[1] >= need1, at most wait_ns of
// device time; on timeout fills the wait-error record `err` (WAIT_PEER).
cudaError_t launch_peer_wait(const unsigned* flags, unsigned need0, unsigned need1, int* err,
                             unsigned long long wait_ns, cudaStream_t st);
// Per-box operations on dense Array3 arrays (yb_hostops.cu): the caller's
// host FieldSet copied to the device as is (element type T = float or double).
struct HostExt {
  int e[6][3];  // extents per component (staggering.hpp:34-39)
};
struct HostBox {
  int xlo, xhi, ylo, yhi, zlo, zhi;
};
template <class T>
struct HostFields {
  T* f[6];         // ex..hz (nullptr where the op does not touch it)
  const T* cd[3];  // Coefficients cdx, cdy, cdz
};
// op 0: update_e_box, 1: update_h_box, 2: zero_box of component `comp`.
template <class T>
cudaError_t launch_host_box(const HostFields<T>& f, const HostExt& x, int op, int comp, const HostBox& b,
                            cudaStream_t st);
// total_energy into scratch[host_energy_scratch_doubles() - 1]; dxyz = dx | dy | dz (double).
template <class T>
cudaError_t launch_host_energy(const HostFields<T>& f, const T* const* prev_h, const HostExt& x,
                               const double* dxyz, int nx, int ny, int nz, double* scratch, cudaStream_t st);
int host_energy_scratch_doubles();

// Halo planes <-> a contiguous exchange buffer: plane q of the list is
// src[q] (or dst[q]) = one padded plane (PX*PY floats); ext holds them in order.
struct HaloList {
  float* plane[12];
  int n;
};
cudaError_t launch_halo_copy(const Geo& g, const HaloList& l, float* ext, bool pack, cudaStream_t st);
cudaError_t launch_fill_value(float* p, long long n, float v, cudaStream_t st);
cudaError_t launch_probes(const Fields& F, const ProbeArgs& pa, float* out, cudaStream_t st);
// weights: x node[nx+1], x cell[nx], y node[ny+1], y cell[ny], z node[nz+1], z cell[nz]
// (local planes); partial: 6*nblk doubles; out: 1 double
constexpr int kEnergyBlocks = 296;
cudaError_t launch_energy(const Geo& g, const Fields& F, const float* const* prev_h, const double* w,
                          double* partial, double* out, cudaStream_t st);
cudaError_t launch_all_equal(const float* a, long long n, int* flag, int num_sms, cudaStream_t st);

}  // namespace yb

namespace yb {
// Caller-memory transfers (yb_xfer.cu): pinned buffers -> cudaMemcpyAsync;
// pageable ones through the pinned staging pipeline (multi-threaded host
// copies overlapped with the DMAs).
bool host_is_pageable(const void* p);
cudaError_t copy_h2d(void* dst, const void* src, size_t n, cudaStream_t st);
cudaError_t copy_d2h(void* dst, const void* src, size_t n, cudaStream_t st);
// The pinned staging ring of yb_xfer.cu, for transfers that stage pieces of their own shape
// (the tile-row readback of yb_run_to_host into pageable memory): hold stage_lock() for the
// whole transfer; stage_acquire(k) waits for chunk k's last DMA (its event, re-created on
// `device`); record stage_event(k) behind the chunk's next DMA. par_for runs fn(0..n-1) over the
// copy-thread pool (the caller's thread included).
constexpr int kStageChunks = 4;
constexpr size_t kStageBytes = size_t(32) << 20;
std::mutex& stage_lock();
cudaError_t stage_init();
void* stage_buf(int k);
cudaError_t stage_acquire(int k, int device);
cudaEvent_t stage_event(int k);
void par_for(int n, const std::function<void(int)>& fn);
}  // namespace yb
