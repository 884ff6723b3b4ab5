/* girih_gpu.h -- C ABI of the B200-native temporally-blocked fp64 stencil sweep.
 *
 * Drop-in boundary for the reference's hot path
 *     girih::run(ProblemState&, long steps, int dw, const WavefrontSpec&,
 *                const ThreadGroupShape&, WavefrontVariant, int n_groups, const RunOptions&)
 * declared at /root/reference/proj/include/girih/engine.hpp:111-115 and implemented at
 * proj/src/engine.cpp:332-418. The reference's callers (verify_once, proj/tools/main.cpp:136;
 * cmd_run, main.cpp:295; make_engine_measure, proj/src/tuner.cpp:220) reach this ABI through
 * the header-only C++ shim include/girih_gpu.hpp (girih::gpu::run), see INTEGRATION.md.
 *
 * Plain pointers and sizes only. Every function returns an int status:
 *   GIRIH_OK (0); GIRIH_EINVAL (-1) <-> std::invalid_argument in the reference
 *   (negative steps, bad kind, extent < 2R+1, negative padding, bad config);
 *   GIRIH_ECUDA / GIRIH_ENCCL / GIRIH_ENOMEM <-> std::runtime_error;
 *   GIRIH_ESTATE <-> std::logic_error (handle misuse).
 * girih_gpu_last_error() returns a thread-local message for the last failure.
 *
 * Host arrays use the reference layout (proj/include/girih/stencil.hpp:31-73): dense
 * [k][j][i] doubles, X = nx + 2R + pad_x, Y = ny + 2R, Z = nz + 2R. Level parity follows
 * stencil.hpp:78-98: time level t lives in u when t is even, in v when t is odd; after a
 * run of T >= 1 steps from t0, the field of parity(t0+T) holds level t0+T and the other
 * field holds level t0+T-1; ghost and pad cells are never written.
 */
#ifndef GIRIH_GPU_H
#define GIRIH_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIRIH_GPU_ABI_VERSION 6

#define GIRIH_OK 0
#define GIRIH_EINVAL (-1)
#define GIRIH_ECUDA (-2)
#define GIRIH_ENCCL (-3)
#define GIRIH_ENOMEM (-4)
#define GIRIH_ESTATE (-5)

/* girih::StencilKind order (stencil.hpp:15) */
#define GIRIH_CONST7PT 0
#define GIRIH_VAR7PT 1
#define GIRIH_CONST25PT 2
#define GIRIH_VAR25PT 3

/* Non-owning view of a host girih::ProblemState (stencil.hpp:83-98). */
typedef struct {
    int kind;
    int nx, ny, nz, pad_x;
    long long t_current;
    double* u;                     /* even time levels */
    double* v;                     /* odd time levels (level -1 seed for const25pt) */
    const double* const* coeffs;   /* n_coeffs coefficient fields (0/7/1/13 by kind) */
    int n_coeffs;
    double cc[5];                  /* scalar coefficients c0..c4 */
} girih_state_view;

/* GPU execution parameters; they replace the CPU engine's (dw, wf, shape, variant, n_groups). */
typedef struct {
    int tb;        /* time steps fused per HBM pass; 0 = tuned/default for the kind */
    int variant;   /* kernel tile variant index (see girih_gpu_variant_info); -1 = default */
    int zchunks;   /* z chunks per tile column; 0 = auto (wave-quantisation model) */
    int ngpus;     /* >1: z-slab decomposition over devices [device, device+ngpus) */
    int exact;     /* 1 = bitwise mode (no FMA contraction); 0 is rejected */
    int device;    /* CUDA device ordinal of the (first) GPU */
    int graphs;    /* >= 0: replay each step's pass sequence as a cached CUDA graph (single-
                      stream handles); -1 = launch passes individually */
    int reserved;  /* >1: emulate that many z-slabs on one device (decomposition tests) */
    int chain;     /* 1 = chain consecutive same-depth passes into one persistent launch whose
                      work units start as soon as their neighbourhood finished the previous pass
                      (single-slab handles); -1 = one launch per pass; 0 = auto (chained for
                      grids of at most 256^3 cells, except var7pt) */
    int tile_order;/* order of the tiles inside a z-chunk row of one-launch-per-pass runs: W > 0 =
                      column strips of W tiles (y fastest inside a strip, so y-neighbour tiles are
                      drawn W apart and share halo rows through L2); -1 = row-major; 0 = auto
                      (strips of 8 for var7pt two-step passes on grids of >= 17 tile columns) */
} girih_gpu_config;

typedef struct {
    double wall_s;          /* host wall time of the call */
    double kernel_s;        /* CUDA-event time of all device work of the step(s) */
    double h2d_s, d2h_s;    /* copy times (girih_gpu_run only) */
    long long lups;         /* nx*ny*nz*steps, interior only (engine.cpp:340) */
    double mlups;           /* lups / kernel_s / 1e6 (girih_gpu_run: lups / wall_s / 1e6) */
    double model_bytes_per_lup; /* algorithmic code balance B1/Tb of the plan */
    int tb_used;            /* largest fused step count of the plan */
    int n_launches;         /* stencil-pass kernel launches */
    double pass_s;          /* summed CUDA-event durations of the stencil-pass launches */
    long long computed_lups;/* LUPs evaluated incl. redundant halo recompute */
    long long h2d_bytes, d2h_bytes;
    int variant_used;
    int zchunks_used;
    int grid_ctas;
    int streamed;           /* girih_gpu_run: 1 = uploads, passes and downloads pipelined along z
                               (skewed task graph; kernel_s is then the whole device span) */
    int n_passes;           /* stencil passes (a chained launch runs several) */
    long long units;        /* work units executed (tile column x z chunk per pass): the GPU
                               counterpart of PerfReport::tiles (engine.hpp:93-98) */
} girih_gpu_report;

/* kernel variant description (compiled tile shapes) */
typedef struct {
    int kind, tb, lx, ly, threads, prefetch;
    int smem_bytes;
    int cluster_y;          /* CTAs per thread-block cluster along y (1 = none): the cluster's
                               CTAs share the fused levels' halo rows through distributed
                               shared memory, or (paced = 1) only run in lockstep */
    int aux_prefetch;       /* coefficient planes fetched ahead */
    int direct_out;         /* 1: output stored from registers (no smem staging + TMA store) */
    int paced;              /* 1: cluster of independent y-neighbour tiles kept on the same z
                               plane by a per-plane cluster barrier (shared rows hit L2) */
    int narrow;             /* > 0: the threads compute only the inner columns of the lx-wide
                               box, and this is the output tile's x halo (output tile width
                               lx - 2 narrow); 0: threads on all lx columns */
} girih_gpu_variant;

const char* girih_gpu_last_error(void);
int girih_gpu_abi_version(void);

/* traits() / stencil_from_name() (proj/src/stencil.cpp:11-17, 41-47) */
int girih_gpu_traits(int kind, int* radius, int* domain_streams, int* flops_per_lup,
                     int* time_order, int* coeff_arrays);
int girih_gpu_kind_from_name(const char* name, int* kind);

/* compiled kernel variants */
int girih_gpu_variant_count(void);
int girih_gpu_variant_info(int index, girih_gpu_variant* out);

/* Open a device-resident state: allocates device buffers and uploads the host view. */
int girih_gpu_open(const girih_state_view* state, const girih_gpu_config* cfg, void** handle);

/* Open a device-resident state initialised ON THE DEVICE with the reference's
 * counter-based generator (init_state, proj/src/stencil.cpp:58-85; values bit-identical).
 * remap = 1 applies the BASELINE.json input remap. */
int girih_gpu_open_seeded(int kind, int nx, int ny, int nz, int pad_x, unsigned long long seed,
                          int remap, const girih_gpu_config* cfg, void** handle);

/* Multi-process z-slabs (one process per GPU): rank 0 creates an NCCL unique id (len >= 128
 * bytes) and shares it; every rank then opens its own slab of the global nx x ny x nz grid on
 * cfg->device, initialised on the device from the global counter-based generator. step()
 * exchanges R*TB halos with ranks rank-1 / rank+1 over NCCL after every pass; download()
 * fills this slab's planes (plus the global ghost planes at the outer slabs) of a global view. */
int girih_gpu_nccl_unique_id(unsigned char* id, int len);
int girih_gpu_open_slab_seeded(int kind, int nx, int ny, int nz, int pad_x, unsigned long long seed,
                               int remap, int rank, int nranks, const unsigned char* nccl_id,
                               const girih_gpu_config* cfg, void** handle);

/* Multi-process halo push over CUDA IPC (open the slab with nccl_id = NULL): each rank exports
 * its buffers and pass flags, passes the blob to its z neighbours (any host transport), then
 * connects to them (NULL for a missing neighbour) and barriers with all ranks. From then on a
 * pass stores its boundary planes straight into the neighbours' halos (peer memory over NVLink)
 * and the ranks order their passes with stream memory operations on each other's flags; no
 * NCCL, no exchange step. */
#define GIRIH_GPU_IPC_BYTES 512
int girih_gpu_ipc_export(void* handle, unsigned char* out, int len);
int girih_gpu_ipc_connect(void* handle, const unsigned char* lower, const unsigned char* upper);

/* Re-upload u, v, coefficients, cc and t_current from a host view of the same shape. */
int girih_gpu_upload(void* handle, const girih_state_view* state);

/* Advance the device state by `steps` (the timed, device-resident hot path). */
int girih_gpu_step(void* handle, long long steps, girih_gpu_report* report);

/* Download u, v and t_current into the view (u/v may be NULL to skip). */
int girih_gpu_download(void* handle, girih_state_view* state);

/* Device-side bitwise compare: field 0 = u, 1 = v, 2 + c = coefficient c
 * of the device state against a host array in state-view layout (X*Y*Z doubles), streamed to the
 * device in z blocks so a large state is checked without downloading it. *n_diff = number of
 * differing cells (ghosts and pad included), *first_index = lowest differing linear index
 * ((k*Y + j)*X + i) or -1. Each slab compares the planes it is authoritative for. */
int girih_gpu_compare(void* handle, int field, const double* host, long long* n_diff,
                      long long* first_index);

/* Download coefficient fields (n pointers, may be NULL entries) and cc[5] (may be NULL). */
/* update_tile (proj/src/engine.cpp:294-330: one tile with a transient thread group, run by the
 * caller once its dependency tiles are complete). GPU counterpart: runs work units
 * [unit_begin, unit_end) of the plan that advances the handle by `steps` steps. Units are
 * numbered pass-major over the plan's passes (*units_total receives the count); a unit is a tile
 * column x z chunk of one pass. Units of one pass are independent (overlapped tiling) and may run
 * in any order and in any pieces; a pass's units need every unit of the earlier passes complete
 * (GIRIH_ESTATE otherwise, as is running a unit twice: the scheduler's double completion,
 * scheduler.cpp:66-69). The state advances by `steps` once every unit has run. Single-slab
 * handles only; the fused depth is the handle's configuration. */
int girih_gpu_update_units(void* handle, long long steps, long long unit_begin, long long unit_end,
                           long long* units_total);

/* Instrumented drop-in call: the counterpart of the reference's RunOptions
 * (proj/include/girih/engine.hpp:100-103, engine.cpp:358-364, 413-416). One device, one launch
 * per pass. `trace_cb` receives one record per work unit (the GPU counterpart of the reference's
 * diamond tile: a tile column x z chunk of one pass) with the CTA that ran it and its
 * %globaltimer start/end, sorted by (pass, unit); `ledger` (steps * nx * ny * nz counts,
 * [t][z][y][x] in interior coordinates, t relative to the call's first step) receives how many
 * times each cell update was produced by the unit that owns it -- exactly once when the tiling,
 * z chunks and slabs partition the grid (UpdateLedger::all_exactly_once, engine.hpp:74-91). */
typedef struct {
    int pass;        /* pass index within the call */
    int unit;        /* work unit within the pass */
    int cta;         /* CTA (block index) that ran it: the reference's thread group */
    int sm;          /* SM it ran on */
    unsigned long long start_ns, end_ns;
} girih_gpu_trace_record;

typedef void (*girih_gpu_trace_fn)(void* ctx, const girih_gpu_trace_record* recs, long long n);

typedef struct {
    girih_gpu_trace_fn trace_cb;  /* NULL: no trace */
    void* trace_ctx;
    long long trace_capacity;     /* records kept (0: 1M); trace_total reports all units */
    long long trace_total;        /* out */
    unsigned int* ledger;         /* NULL: no ledger; else steps * nx * ny * nz counts (out) */
} girih_gpu_run_options;

/* girih_gpu_run with instrumentation (opts NULL or empty: exactly girih_gpu_run) */
int girih_gpu_run_ex(girih_state_view* state, long long steps, const girih_gpu_config* cfg,
                     girih_gpu_report* report, girih_gpu_run_options* opts);

/* Device-side digest of a whole field (0 = u, 1 = v, 2 + c = coefficient c), ghosts and pad
 * included: FNV-1a over the FNV-1a hashes of every allocated row in (k, j) order (one GPU
 * thread per row). A checksum of checksums of the full state that needs no download; the
 * oracle computes the same function on host arrays (orc_row_digest). */
int girih_gpu_row_digest(void* handle, int field, unsigned long long* digest);

int girih_gpu_download_coeffs(void* handle, double* const* coeffs, int n, double* cc);

int girih_gpu_get_t(void* handle, long long* t_current);
int girih_gpu_set_config(void* handle, const girih_gpu_config* cfg);
int girih_gpu_close(void* handle);

/* open + step + download + close: the drop-in for girih::run (engine.hpp:113-115). */
int girih_gpu_run(girih_state_view* state, long long steps, const girih_gpu_config* cfg,
                  girih_gpu_report* report);

/* Host-side pass planner (exposed for tests): splits `steps` into passes of at most tb
 * fused steps and assigns buffers. Buffer ids: 0 = u, 1 = v, 2 = even scratch,
 * 3 = odd scratch; -1 = none. Arrays have room for max_passes entries. */
int girih_gpu_plan(int kind, long long t0, long long steps, int tb, int max_passes,
                   int* n_passes, int* pass_tb, int* pass_src, int* pass_src_prev,
                   int* pass_dst, int* pass_dst_penult);

/* GPU analogue of the analytic models (proj/src/models.cpp:12-84; cache_block_size, code_balance,
 * roofline): tile geometry, shared-memory footprint per CTA (the counterpart of Eq. 2's C_S),
 * redundant halo recompute, code balance (algorithmic B1/Tb and the no-L2-reuse bound) and the
 * roofline min(HBM*Tb/B1, FP64/(DP ops*redundancy)) of one (kind, grid, tb, variant). tb = 0 /
 * variant = -1 select the defaults; hbm_gbs / fp64_ops <= 0 select the measured B200 peaks
 * (6558.7 GB/s copy, 18.59e12 DADD/DMUL ops/s). Host-only (no device needed). */
typedef struct {
    int tb, variant, lx, ly, ox, oy, threads;
    int smem_bytes;          /* dynamic shared memory per CTA */
    int ctas_per_sm;         /* resident CTAs per SM allowed by shared memory and threads */
    int tiles_x, tiles_y, zchunks, zc_len;
    double redundancy;       /* evaluated level-cell updates per useful LUP */
    double code_balance;     /* algorithmic bytes/LUP, B1/Tb */
    double code_balance_no_l2; /* bytes/LUP if every tile re-streamed its whole box from HBM */
    double hbm_mlups, fp64_mlups, roofline_mlups;
} girih_gpu_model_out;
int girih_gpu_model(int kind, int nx, int ny, int nz, int tb, int variant, double hbm_gbs,
                    double fp64_ops, girih_gpu_model_out* out);

/* z-slab decomposition used by multi-GPU handles: slab g of nslabs owns interior planes
 * [*z0, *z1) (0-based interior z) and carries *hz halo planes per side (R * max fused depth). */
int girih_gpu_slab_layout(int kind, int nz, int nslabs, int g, int* z0, int* z1, int* hz);

/* On-device auto-tuner (replaces girih::tune, proj/src/tuner.cpp:146-210): hill-climbs
 * (tb, variant, zchunks) with CUDA-event timing and adaptive test sizing on the handle's
 * own state (the state is restored afterwards). Writes the best config into *best. */
int girih_gpu_tune(void* handle, int max_tb, girih_gpu_config* best, double* best_mlups,
                   int* n_measured);

/* Release the device memory the library keeps cached between handles (freed state buffers are
 * reused by the next open/run of the same size instead of cudaMalloc/cudaFree per call). */
int girih_gpu_trim(void);

/* pinned host memory helpers (for H2D/D2H at full PCIe rate) */
int girih_gpu_host_alloc(size_t bytes, void** ptr);
int girih_gpu_host_free(void* ptr);

/* interior_checksum (proj/src/stencil.cpp:129-146) of the current level of a host view */
int girih_gpu_interior_checksum(const girih_state_view* state, unsigned long long* out);

/* measured FP64 rates on `device` (ops/s of separate DADD/DMUL and of DFMA) */
int girih_gpu_fp64_peak(int device, double* dadd_dmul_ops_per_s, double* dfma_flops_per_s);

/* device properties (SM count, name) */
int girih_gpu_device_info(int device, int* sm_count, char* name, int name_len);

#ifdef __cplusplus
}
#endif

#endif /* GIRIH_GPU_H */
