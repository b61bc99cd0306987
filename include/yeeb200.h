/*
 * yeeb200.h — C-ABI of libyeeb200.so, the B200 (sm_100a) implementation of
 * the reference yeeblock Standard leapfrog step (arXiv 1301.4539 hot path).
 *
 * Plain C: opaque handle, plain pointers and sizes, int status codes. The
 * C++ shim include/yeeb200/yeeblock.hpp maps the codes back onto the
 * reference's exception types and re-exposes the reference API names.
 *
 * Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj/include/yeeblock/).
 *
 * Field arrays crossing this boundary use the reference's dense Array3
 * layout of each component: extents from staggering.hpp:34-39
 *   ex nx x (ny+1) x (nz+1)   ey (nx+1) x ny x (nz+1)   ez (nx+1) x (ny+1) x nz
 *   hx (nx+1) x ny x nz       hy nx x (ny+1) x nz       hz nx x ny x (nz+1)
 * and index (k*ny_c + j)*nx_c + i (array3.hpp:104-107). Per-cell
 * coefficient arrays are nx*ny*nz in the same cell order.
 *
 * Threading: one host thread per handle at a time (like FieldSet /
 * Simulation). Work is enqueued on the handle's CUDA stream;
 * calls that return data to the host synchronise that stream.
 */
#ifndef YEEB200_H
#define YEEB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define YB_ABI_VERSION 5

/* Status codes. The shim maps INVALID_ARGUMENT -> std::invalid_argument,
 * OUT_OF_RANGE -> std::out_of_range, the rest -> std::runtime_error. */
enum {
  YB_OK = 0,
  YB_INVALID_ARGUMENT = 1,
  YB_OUT_OF_RANGE = 2,
  YB_RUNTIME_ERROR = 3,
  YB_CUDA_ERROR = 4
};

/* Components, in the reference's canonical order (staggering.hpp:12). */
enum { YB_EX = 0, YB_EY, YB_EZ, YB_HX, YB_HY, YB_HZ };

/* Per-cell coefficient selectors (extension; the reference has none). */
enum { YB_CA = 0, YB_CB = 1, YB_DA = 2, YB_DB = 3 };

/* Step implementations. A zero-initialised yb_desc selects YB_VARIANT_TB2,
 * the fastest path (ABI 3; ABI 2 had FUSED = 0 and TB2 = 2). */
enum {
  YB_VARIANT_TB2 = 0,   /* temporal blocking: two full steps per sweep (odd remainder: FUSED) */
  YB_VARIANT_NAIVE = 1, /* one thread per DoF, separate E/PEC/source/H launches */
  YB_VARIANT_FUSED = 2, /* one z-march sweep per step: TMA-staged planes, E+H fused */
  YB_VARIANT_TB4 = 3    /* temporal blocking: four full steps per sweep (remainder: TB2 / FUSED);
                           single domain; the depth-8 point of the temporal-depth sweep */
};

typedef struct yb_sim yb_sim;

typedef struct {
  int nx, ny, nz; /* cells per axis (GridSpec, grid.hpp:17-43); nz = this slab's depth */
  int device;     /* CUDA device ordinal */
  int variant;    /* YB_VARIANT_* (0 = TB2, the default) */
  int zchunk;     /* fused: z planes per work item; 0 = auto */
  int z_offset;   /* z-slab mode: global index of local cell plane 0 (0 otherwise) */
  int nz_global;  /* z-slab mode: global cell count along z (0 = nz, single domain) */
  int reserved[4];
} yb_desc;

typedef struct {
  int64_t step_index;      /* completed steps (FieldSet::step_index, fields.hpp:24) */
  int64_t steps;           /* steps advanced through this handle */
  int64_t kernel_launches; /* kernels launched by yb_advance so far */
  double main_kernel_ms;   /* summed device time of the main sweep kernel (timing on) */
  int64_t main_kernel_timed;
  int n_cell_arrays;       /* per-cell coefficient arrays read by the step (0..4) */
  int variant;
  int stages;              /* fused: TMA ring depth */
  int grid_x, grid_y, grid_z;
  int zchunk;
  double bytes_per_cell_update; /* algorithmic HBM bytes per cell-update, one sweep */
  size_t device_bytes;     /* device memory held by the handle */
  int halo_depth;          /* z-slab mode: ghost planes refreshed per exchange = steps per exchange */
  int quiescent_skip;      /* yb_set_quiescent_skip state */
  int64_t skipped_items;   /* work items skipped as quiescent (RunStats::skipped_tiles analogue) */
  int64_t streamed_readbacks; /* yb_run_to_host calls whose readback overlapped the run */
  int64_t streamed_uploads;   /* yb_run_streamed calls whose upload overlapped the run */
} yb_info;

/* Last error message of the calling thread ("" if none). */
const char* yb_last_error(void);
int yb_abi_version(void);

/* Simulation<Real> ctor (runner.hpp:208-234) minus the CPU tiling: allocates
 * device-resident padded SoA fields (zeroed, step_index 0). Coefficients
 * start as Ca = Da = 1, Cb/Db = per-axis arrays filled with 0 (call
 * yb_set_axis_coeffs, the build_coefficients replacement). */
int yb_create(const yb_desc* desc, yb_sim** out);
int yb_destroy(yb_sim* sim);

/* Coefficients<Real>{cdx,cdy,cdz} (grid.hpp:79-103): the reference's one
 * coefficient set, used by both curls where no per-cell Cb/Db is set. */
int yb_set_axis_coeffs(yb_sim* sim, const float* cdx, const float* cdy, const float* cdz);

/* Per-cell coefficients (extension). which = YB_CA/YB_DA: `cells` (nx*ny*nz)
 * or NULL to use the scalar `uniform`. which = YB_CB/YB_DB: `cells` or NULL
 * to fall back to the per-axis arrays. Update forms (reference operand
 * order, kernels.hpp:27-63):
 *   e = Ca*e + (Cb*(a-b) - Cb*(c-d)),  h = Da*h + (Db*(a-b) - Db*(c-d)).
 * An uploaded array whose values are all equal is stored as a uniform
 * value (Ca/Da scalar; Cb/Db as a constant per-axis set) - bit-identical,
 * one array fewer to stream. */
int yb_set_cell_coeffs(yb_sim* sim, int which, const float* cells, float uniform);

/* Device-side generation of the pinned seeded medium (include/yeeb200_inputs.h):
 * eps_seed < 0 -> eps = 1; sigma_seed < 0 -> sigma = 0. With sigma = 0 the
 * Ca/Da arrays are exactly 1 and Db exactly S, so only Cb is stored. */
int yb_generate_medium(yb_sim* sim, int64_t eps_seed, int64_t sigma_seed);

/* Host-side generators of the same pinned inputs, for callers that feed the
 * drop-in from host memory (no handle, no GPU needed). Any of the four
 * coefficient outputs may be NULL. Dense reference layouts. */
int yb_host_medium(int nx, int ny, int nz, int64_t eps_seed, int64_t sigma_seed, float* ca,
                   float* cb, float* da, float* db);
int yb_host_field(int nx, int ny, int nz, uint64_t seed, int comp, float* dense);
/* The same for the z-slab [z_offset, z_offset+nplanes) of a grid with
 * nz_global planes: `nplanes` dense planes of the component (clipped to its
 * global extent) / `nplanes` cell planes of the medium (z_offset may be
 * negative; planes outside the grid get clamped copies). */
int yb_host_field_slab(int nx, int ny, int nz_global, int z_offset, int nplanes, uint64_t seed,
                       int comp, float* dense);
int yb_host_medium_slab(int nx, int ny, int nz_global, int z_offset, int nplanes,
                        int64_t eps_seed, int64_t sigma_seed, float* ca, float* cb, float* da,
                        float* db);

/* FieldSet readout/writeback (fields.hpp:21-67). Dense reference layout. */
int yb_upload_field(yb_sim* sim, int comp, const float* dense);
int yb_download_field(yb_sim* sim, int comp, float* dense);
/* All six components (Ex, Ey, Ez, Hx, Hy, Hz) in one call: the host<->device
 * copies run back to back while the dense<->padded layout conversion of the
 * previous component overlaps them; one synchronisation at the end (the host
 * buffers may be reused when the call returns). */
int yb_upload_fields(yb_sim* sim, const float* const* dense6);
/* Several per-cell coefficient arrays in one call (which[i] in CA..DB, each
 * at most once, cells[i] non-null): the copies run back to back with one
 * synchronisation for their uniformity checks; otherwise as n calls of
 * yb_set_cell_coeffs(which[i], cells[i], 0). */
int yb_set_cell_coeffs_n(yb_sim* sim, int n, const int* which, const float* const* cells);
int yb_download_fields(yb_sim* sim, float* const* dense6);
/* Simulation::run followed by the FieldSet readout (runner.hpp:243-266 +
 * fields.hpp:21-67): advance nsteps, then leave all six components in the
 * dense host buffers — the drop-in form of `sim.run(n); sim.fields()`.
 * With page-locked buffers and the two-step kernel on a single domain
 * (no probes, no quiescent skip, nsteps >= 4) the readback overlaps the run:
 * the last multi-sweep launch hands its items out along y-skewed diagonals,
 * and each tile row's device->host copies start as soon as it finished its
 * last sweep. Otherwise it is yb_advance + yb_download_fields. Same result
 * either way (bit-identical). */
int yb_run_to_host(yb_sim* sim, int64_t nsteps, float* const* dense6);
/* run_simulation's whole host flow in one call (runner.hpp:349-362: construct
 * from a GridSpec + state, run, read the FieldSet back): upload ncoef per-cell
 * coefficient arrays (which[] = YB_CA..YB_DB, dense nx*ny*nz each) and, when
 * in6 is not NULL, the six initial field components; advance nsteps; leave
 * all six components in out6. in6 == NULL runs from the handle's current
 * state (the zero FieldSet of a fresh handle). With page-locked buffers on a
 * single domain with the two-step kernel (no probes, no quiescent skip, an
 * even nsteps in 8 .. 2048) both transfers overlap the run: the copies go up
 * tile row by tile row and the one multi-sweep launch hands out its first
 * sweeps along the mirrored y-skewed diagonals, each first-sweep item
 * starting once its rows have landed (per-row words the copy stream writes,
 * cuStreamWriteValue32), and its last sweeps as yb_run_to_host does. The
 * arrays are stored as given (no uniformity compression). Otherwise it is
 * yb_set_cell_coeffs_n + yb_upload_fields + yb_run_to_host. Same result either
 * way (bit-identical). */
int yb_run_streamed(yb_sim* sim, int64_t nsteps, int ncoef, const int* which, const float* const* cells,
                    const float* const* in6, float* const* out6);
/* FieldSet::zero() (fields.hpp:60-63) and seeded init (yeeb200_inputs.h). */
int yb_zero_fields(yb_sim* sim);
int yb_fill_fields(yb_sim* sim, uint64_t seed);
int yb_set_step_index(yb_sim* sim, int64_t step_index);
int yb_get_step_index(yb_sim* sim, int64_t* step_index);

/* Soft point source on one E DoF (SourceSpec + inject_current,
 * source.hpp:33-68): comp(i,j,k) += table[step] at each step < n, after
 * Ampere and PEC, before Faraday. Position must be strictly interior
 * (SourceSpec::validate, source.hpp:43-55). At most YB_MAX_SOURCES. */
#define YB_MAX_SOURCES 8
int yb_add_source(yb_sim* sim, int comp, int i, int j, int k, const float* table, int64_t n);
int yb_clear_sources(yb_sim* sim);

/* Point probes (ProbeSpec + sample_probes, probe.hpp:14-51): after every
 * completed step t with t % stride == 0 the probe's value is recorded on the
 * device (no full-field readback). Positions index the component's own
 * extents (ProbeSpec::validate). Two-step sweeps are split into single steps
 * where a probe fires in between (the reference suspends pairing likewise,
 * runner.hpp:279-285). Single-domain handles only. At most YB_MAX_PROBES. */
#define YB_MAX_PROBES 64
int yb_set_probes(yb_sim* sim, int n, const int* comp, const int* i, const int* j, const int* k,
                  const int* stride);
/* Moves up to `capacity` recorded samples (oldest first) to the host:
 * step (completed steps), probe index, value; *count = number returned. */
int yb_read_probes(yb_sim* sim, int64_t* steps, int* probe, float* values, int64_t capacity,
                   int64_t* count);

/* Leapfrog energy invariant (total_energy + HSnapshot, fields.hpp:68-146).
 * yb_snapshot_h copies the current H (the reference's HSnapshot); after
 * advancing, yb_total_energy returns sum_E V*E^2 + sum_H V*Hprev*Hnow with
 * V the dual/primal cell volumes from the spacings dx[nx], dy[ny],
 * dz[nz_global] (NULL = unit spacing), accumulated in double (deterministic;
 * summation order differs from the reference's serial loop). On a z-slab the
 * sum covers the planes the slab owns (sum over ranks for the total). */
int yb_snapshot_h(yb_sim* sim);
int yb_total_energy(yb_sim* sim, const double* dx, const double* dy, const double* dz, double* energy);

/* Quiescent skip (runner.hpp:60-73, :287-313; RunOptions::quiescent_skip):
 * when on, a sweep work item whose whole input box is exactly +0 in both
 * state buffers and touches no active source is not computed (its result is
 * +0 bit for bit). Tracked as one bit per (tile, plane), set once the
 * tile-plane may hold a nonzero value; rebuilt by a device scan after any
 * host-side change of the state. Results are identical with it on or off.
 * Default off. The naive variant ignores it. */
int yb_set_quiescent_skip(yb_sim* sim, int on);

/* Simulation::run(n) time loop (runner.hpp:243-266) with the Standard step
 * (schedule.hpp:171-210): advances step_index by n. Asynchronous on the
 * handle's stream. */
int yb_advance(yb_sim* sim, int64_t nsteps);
int yb_synchronize(yb_sim* sim);
/* yb_advance bracketed by CUDA events on the handle's stream; *ms = elapsed. */
int yb_advance_timed(yb_sim* sim, int64_t nsteps, float* ms);

/* Range operations (kernels.hpp:129-155), in place on the current state.
 * box = {xlo,xhi,ylo,yhi,zlo,zhi} in node index space, must lie inside
 * [0,nx]x[0,ny]x[0,nz] (detail::check_range, kernels.hpp:118-122) else
 * YB_OUT_OF_RANGE. NULL box = whole domain. */
int yb_apply_ampere_range(yb_sim* sim, const int* box);
int yb_apply_faraday_range(yb_sim* sim, const int* box);
int yb_apply_pec_boundary(yb_sim* sim);

/* field_digest (fields.hpp:151-166): FNV-1a-64 over the dense Ex..Hz bytes. */
int yb_field_digest(yb_sim* sim, uint64_t* out);

/* z-slab decomposition (desc.nz_global > desc.nz; FUSED or TB2 variant). The
 * slab owns global cell planes [z_offset, z_offset+nz). Ghost planes are
 * refreshed from the neighbours every yb_info.halo_depth = d steps (d = 1
 * FUSED, 2 TB2): exchange, then yb_advance(sim, d).
 *   side 0 (bottom, rank below): send my planes 0..d-1 (all six components);
 *                                receive -> my ghosts -d (hx,hy), -d+1..-1 (all)
 *   side 1 (top, rank above):    send my planes nz-d (hx,hy), nz-d+1..nz-1 (all);
 *                                receive -> my ghosts nz..nz+d-1 (all)
 * Buffers are device memory of yb_halo_bytes(sim, side, 0|1) bytes
 * (0: what this side sends, 1: what it receives); plane = PX*PY floats. A
 * slab's dense field arrays are the local part of the global Array3 (node-z
 * components carry nz+1 planes; the top one belongs to the rank above unless
 * this is the global top). Per-cell coefficient uploads in slab mode carry
 * nz+4 cell planes: global planes z_offset-2 .. z_offset+nz+1 (planes outside
 * the grid are ignored). Axis coefficient cdz is the GLOBAL array.
 * pack / unpack are enqueued on the handle's stream: on a caller stream
 * (yb_set_stream) they are stream-ordered and return at once, so a
 * transport enqueued on the same stream (e.g. NCCL through torch) needs no
 * host synchronisation; on the handle's own stream they complete before
 * returning. */
int yb_halo_bytes(yb_sim* sim, int side, int receive, size_t* bytes);
/* Split sweep for overlapping the exchange with compute: yb_advance_begin(n)
 * (n <= halo depth) launches the sweep over the slab's boundary planes
 * [0, n) and [nz-n, nz) only; yb_halo_pack then reads those NEW planes, so
 * the transfer can run while yb_advance_end launches the interior planes and
 * completes the n steps; yb_halo_unpack after yb_advance_end. Bit-identical
 * to yb_advance(n). No probes; not the NAIVE variant. */
int yb_advance_begin(yb_sim* sim, int64_t nsteps);
int yb_advance_end(yb_sim* sim);

/* Direct halo push over peer memory (NVLink P2P between GPUs; CUDA IPC
 * between processes, or plain pointers within one process) instead of
 * pack + NCCL + unpack. Setup: yb_peer_export writes yb_peer_handle_bytes()
 * bytes of IPC handles (the state buffers and a flag block) for the
 * neighbour to yb_peer_open (side 0: the slab below, 1: above; peer_nz its
 * depth); within one process yb_peer_link takes the neighbour's handle.
 * Per exchange: yb_peer_push copies this slab's d = halo-depth boundary
 * planes (the new ones while a split sweep is in flight, else the current
 * state's) into the neighbours' ghost planes and then publishes a counter in
 * their flag words (overlap = 1: on a side stream, concurrent with the
 * interior sweep); yb_peer_wait makes this handle's stream wait (on the
 * device) until both neighbours have pushed as often as it has. Schedule:
 * push; then per exchange: wait, yb_advance_begin(d), push, yb_advance_end.
 * A wait that never completes gives up after ~15 s and yb_synchronize reports
 * YB_RUNTIME_ERROR. Neighbours store into this slab's memory: synchronise
 * all ranks before yb_destroy. */
size_t yb_peer_handle_bytes(void);
int yb_peer_export(yb_sim* sim, void* handles);
int yb_peer_open(yb_sim* sim, int side, const void* handles, int peer_nz);
int yb_peer_link(yb_sim* sim, int side, yb_sim* other);
int yb_peer_push(yb_sim* sim, int overlap);
int yb_peer_wait(yb_sim* sim);
/* One exchange period over peer memory. TB2, nsteps = 2: ONE launch — a
 * two-step sweep whose boundary-plane stores also land in the neighbours'
 * ghost planes (the exchange fused into the compute kernel); its bottom / top
 * z-chunk items run first, wait in-kernel for the neighbour's previous period
 * and the last of them signals this one (separate wait / signal launches
 * when the grid's first or last z-chunk is under two planes). nsteps = 1:
 * wait, split sweep, push. Start a run with one yb_peer_push of the current
 * state. */
int yb_peer_step(yb_sim* sim, int64_t nsteps);
/* Chained exchange periods: nsteps (even) / 2 periods in ONE persistent
 * two-step launch — per sweep, the bottom / top z-chunk items wait in-kernel
 * for the neighbour's previous sweep, store their boundary planes into its
 * ghost planes and signal, while the sweeps follow each other through
 * device-side neighbourhood counts (no launch gap or wave tail between
 * periods). sims[0..n): n = 1, one rank's slab (its neighbours make the same
 * call on their GPUs); n = 2..8, linked slabs of ONE device run in the same
 * launch (the one-GPU emulation of n ranks — never separate launches that
 * wait on each other). Two-step variant, no probes; starts, like
 * yb_peer_step, after one yb_peer_push of the current state. Extension (the
 * reference has no multi-GPU path). */
int yb_peer_run(yb_sim* const* sims, int n, int64_t nsteps);
int yb_halo_pack(yb_sim* sim, int side, void* dst_device);
int yb_halo_unpack(yb_sim* sim, int side, const void* src_device);

/* Per-box operations on a caller's FieldSet<Real> held in HOST memory: the
 * reference's free functions, for either precision (the reference is
 * templated on Real; its own unit tests run in double). The components the
 * operation reads are copied to device `device`, it runs as per-DoF kernels
 * in the reference's operand order (bit-identical in fp32 and fp64), and the
 * components it writes are copied back. No handle; synchronous. For the
 * device-resident fp32 time loop use a yb_sim handle instead.
 *   dense6: Ex..Hz arrays (dense Array3 layout, element type dtype)
 *   cd3:    Coefficients cdx[nx], cdy[ny], cdz[nz] (dtype; unused by ZERO / PEC)
 *   box:    {xlo,xhi,ylo,yhi,zlo,zhi} (IndexBox; unused by PEC)
 *   op:     YB_OP_UPDATE_E  update_e_box(f, c, comp, box)   kernels.hpp:78-88
 *           YB_OP_UPDATE_H  update_h_box(f, c, comp, box)   kernels.hpp:92-101
 *           YB_OP_ZERO      zero_box(f, comp, box)          kernels.hpp:104-111
 *           YB_OP_AMPERE    apply_ampere_range(f, c, box)   kernels.hpp:129-135
 *           YB_OP_FARADAY   apply_faraday_range(f, c, box)  kernels.hpp:138-144
 *           YB_OP_PEC       apply_pec_boundary(f)           kernels.hpp:147-155
 * Boxes outside the ranges the reference accepts -> YB_OUT_OF_RANGE with the
 * reference's message. */
enum { YB_F32 = 0, YB_F64 = 1 };
enum { YB_OP_UPDATE_E = 0, YB_OP_UPDATE_H, YB_OP_ZERO, YB_OP_AMPERE, YB_OP_FARADAY, YB_OP_PEC };
int yb_fs_apply(int device, int dtype, int nx, int ny, int nz, void* const* dense6, const void* const* cd3, int op,
                int comp, const int* box);
/* total_energy(g, f, prev_h) (fields.hpp:116-146) of a host FieldSet and
 * HSnapshot (prev_h3 = Hx, Hy, Hz), spacings dx/dy/dz (NULL = 1), double
 * accumulation on the device (deterministic; summation order differs from
 * the reference's serial loop). */
int yb_fs_total_energy(int device, int dtype, int nx, int ny, int nz, const void* const* dense6,
                       const void* const* prev_h3, const double* dx, const double* dy, const double* dz,
                       double* energy);

/* Work on a caller-owned stream (e.g. torch.cuda.current_stream()); NULL
 * restores the handle's own stream. */
int yb_set_stream(yb_sim* sim, void* cuda_stream);
/* Accumulate per-launch device time of the main sweep kernel into yb_info. */
int yb_set_kernel_timing(yb_sim* sim, int on);
int yb_get_info(yb_sim* sim, yb_info* info);

#ifdef __cplusplus
}
#endif

#endif /* YEEB200_H */
