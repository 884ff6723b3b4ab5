// zwave.cuh -- the temporally-blocked z-wavefront stencil pass for sm_100a.
//
// One launch advances a z-slab (or the whole grid) by TB time steps in a single HBM pass.
// It is the B200 counterpart of the reference's multi-core wavefront diamond engine
// (proj/src/engine.cpp:203-260): there a thread group shares one cache block and sweeps z
// with a pipelined wavefront; here a CTA owns an (x,y) tile column and streams its z-planes
// through shared memory:
//
//   * level 0 (the input time level) arrives plane by plane by TMA (cp.async.bulk.tensor,
//     box LX x LY x 1) into a ring of NR0 = R+1+P planes completed on mbarriers, P planes
//     ahead of use -- the z-wavefront; thread 0 issues the loads, warp 1 the output stores;
//   * the time-invariant coefficient fields (one contiguous [c][k][j][i] block) arrive by ONE
//     4-D TMA per plane (box AX x AY x 1 x NC, the level-1 area) into an aux ring deep enough
//     that level s re-uses the plane level 1 fetched (s-1)*R iterations earlier -- each
//     coefficient byte crosses HBM once per pass, not once per fused step (var7pt TB=2 carries
//     level 1's coefficients to level 2 in registers instead); const25pt's level t0-1 field
//     rides in the same aux ring;
//   * a thread owns the same x-pairs of cells at every level (the rows [R, LY-R) of the tile);
//     level s (1..TB) of plane k_s = j - s*R is computed at global iteration j from level
//     s-1: x/y neighbours from the level-(s-1) centre plane in smem, z neighbours k_s-R ..
//     k_s+R-1 from the thread's own register queue, k_s+R from the value it produced one
//     level earlier in the same iteration;
//   * levels 1..TB-1 keep rings of R+1 centre planes; level TB goes to a staging plane and
//     out by a TMA store clipped to the interior (an odd nx's last column is stored directly);
//   * the tile shrinks by R per side per level (overlapped / trapezoid tiling in x and y,
//     and in z at z-chunk boundaries), so no inter-CTA synchronisation exists inside a pass;
//     the x halo is H or H+1 so that every TMA box starts on a 16-byte boundary;
//   * inner-columns-only tiles (ZwaveConfig::NARROW): the box is 64 + 2 XO columns wide and the
//     threads sit on its inner 64 columns, so a single-step tile outputs all 64 thread columns
//     (tiles divide 256 / 512 exactly, no thread computes a halo column) and the fused var7pt
//     tile 62 instead of 60;
//   * work units (tile, z-chunk) are drawn dynamically in z-chunk-major order, which keeps
//     neighbouring tiles within about a chunk of each other in z so shared halo rows are
//     still in L2.
//
// One __syncthreads per z-plane orders every cross-thread smem dependency: all values a
// level reads from smem were produced at least one iteration earlier.
//
// Bitwise parity with the oracle (proj/src/stencil.cpp:115-127): every point expression
// is evaluated with the operand association of proj/include/girih/kernels.hpp:31-85 using
// __dmul_rn/__dadd_rn/__dsub_rn (no FMA contraction, CMakeLists.txt:24-25 -ffp-contract=off),
// ghost cells of intermediate levels take the value of the parity-(t0+s) field
// (stencil.hpp:78-82, kernels.hpp:25-26), and the const25pt leapfrog reads level s-2 at
// the centre (kernels.hpp:50-52).
#pragma once

#include <cuda.h>
#include <cstdint>
#include <type_traits>

#ifndef GIRIH_CHAIN_MINB_DROP
#define GIRIH_CHAIN_MINB_DROP 0  // A/B: chained kernels one resident CTA fewer (more registers)
#endif
#ifndef GIRIH_PHZ
#define GIRIH_PHZ 1  // single-pass const25pt: z queue rotated by renaming (see PHZ)
#endif
#ifndef GIRIH_PHZ_ALL
#define GIRIH_PHZ_ALL 0  // A/B: PHZ for every single-step radius-4 kernel
#endif
#ifndef GIRIH_ZPS
#define GIRIH_ZPS 1  // single-step radius-4 passes: z+ neighbours from the level-0 ring
#endif
#ifndef GIRIH_PHQ
#define GIRIH_PHQ 0  // A/B: single-pass var7pt TB = 2 rotates its z and coefficient queues by renaming (PHQ: -13%)
#endif
#ifndef GIRIH_ZPS_ALL25
#define GIRIH_ZPS_ALL25 0  // A/B: ZPS for single-pass const25pt without PHZ
#endif
#ifndef GIRIH_LOCK
#define GIRIH_LOCK 0  // lockstep pacing compiled in (PassParams::lock; A/B builds only: its
                      // producer state cost the bench kernel a spill and 2-4%)
#endif
#ifndef GIRIH_PACE_LAG
#define GIRIH_PACE_LAG 2  // PACE clusters: planes a CTA may run ahead of its y-neighbours
#endif
#ifndef GIRIH_IPC_FLAGS
#define GIRIH_IPC_FLAGS 1  // single-pass kernels signal IPC neighbours after their boundary units
#endif
#ifndef GIRIH_UORDER
#define GIRIH_UORDER 1  // unit orders other than z-chunk-major (A/B switches GIRIH_UGROUP/USTRIP)
#endif
#ifndef GIRIH_XSHFL
#define GIRIH_XSHFL 1  // x neighbours by warp shuffle where measured faster (see XSHFL)
#endif

namespace girih_gpu {

enum { K_CONST7 = 0, K_VAR7 = 1, K_CONST25 = 2, K_VAR25 = 3 };

template <int KIND> struct KindTraits;
template <> struct KindTraits<K_CONST7> { static constexpr int R = 1, NC = 0, LEAP = 0; };
template <> struct KindTraits<K_VAR7> { static constexpr int R = 1, NC = 7, LEAP = 0; };
template <> struct KindTraits<K_CONST25> { static constexpr int R = 4, NC = 1, LEAP = 1; };
template <> struct KindTraits<K_VAR25> { static constexpr int R = 4, NC = 13, LEAP = 0; };

// Everything one pass needs; passed by value as a __grid_constant__ parameter.
struct PassParams {
    const double* src_prev;  // const25pt: buffer holding level t0-1 (read at the centre only)
    double* dst_final;       // level t0+TB   (interior cells of the output tiles)
    double* dst_penult;      // level t0+TB-1 (same cells) or nullptr
    const double* ghost[2];  // pristine fields by parity (u = even, v = odd): ghost values
    const double* coeff[13]; // coefficient fields (device layout)
    double cc[5];
    int parity0;             // parity of t0
    int nx, ny;              // interior extents
    int X, Y;                // allocated extents of a row / of a plane (rows)
    int pitch;               // device row pitch (elements)
    int off;                 // element offset of allocated x = 0 inside a device row
    long long plane;         // elements per plane = pitch * Y
    int Zloc;                // planes in the local buffer
    int zoff;                // global allocated plane index of local plane 0
    int nzg;                 // global interior z extent
    int tiles_x, tiles_y;    // tile grid
    int nzc, zc_len;         // z chunks per tile column and output planes per chunk
    int zout_lo, zout_hi;    // local output planes [lo, hi)
    int work_base;           // value of *work when this pass started (cumulative per step)
    int oz0;                 // local plane of the output store map's z = 0 (the slab's zout_lo)
    int units;               // tiles_x * tiles_y * nzc
    int unit0, unit_n;       // single-pass launches run units [unit0, unit0 + unit_n)
    int* work;               // dynamic unit counter (zeroed before every launch)
    unsigned long long* ptrace;  // optional per-iteration phase clocks of CTA 0 (debug)
    int hx, ox;              // x halo (H or H+1) and output tile width LX - 2*hx: TMA needs the
                             // innermost box coordinate 16-byte aligned (even for fp64)
    int xorg;                // allocated x of local column 0 of tile column 0: R - hx, or one less
                             // when that makes the TMA origins even (output-only tiles with an odd
                             // halo: the first tile's first output column then sits on the ghost
                             // column and is masked like any ghost cell)
    // Halo push (single-process z-slabs): the output cells of this slab's bottom / top push_hz
    // own planes are also stored straight into the lower / upper neighbour's halo planes (peer
    // memory over NVLink, or the same device for emulated slabs), so no exchange step follows
    // the pass. A neighbour cell = its base + (local plane k * plane + push_*_off) + column.
    double* push_dn_final;
    double* push_up_final;
    double* push_dn_penult;
    double* push_up_penult;
    long long push_dn_off, push_up_off;
    int push_hz;
    // Instrumentation (girih_gpu_run_ex, the reference's RunOptions, engine.hpp:100-103; off
    // when null): per-unit trace records appended at trace[4 * atomicAdd(trace_n, 1)] =
    // {pass << 32 | unit, cta << 32 | sm, start ns, end ns} (%globaltimer), and the ledger of
    // owned cell updates [step][z][y][x] (interior coordinates), +1 per output cell and level.
    unsigned long long* trace;
    unsigned long long* trace_n;
    long long trace_cap;
    int trace_pass;
    unsigned* ledger;
    int ledger_t;  // step index (from the start of the call) of this pass's level 1
    // Lockstep (single-pass, non-cluster launches; off when lock is null). The CTAs of a
    // persistent grid drift apart under dynamic unit drawing until neighbouring tiles stream
    // the same planes tens of iterations apart, beyond the ~13 iterations a plane stays in L2,
    // and every shared halo row then comes from DRAM twice. Each CTA's load producer counts its
    // issued planes in blocks of lock_blk and may not start block m before every CTA of the
    // grid has reached block m - lock_slack: *lock counts block arrivals from lock_base on
    // (relaxed atomics: pure pacing, no data is exchanged). A CTA out of units adds the
    // remainder of its 2^32 arrivals, so the rest never wait for it. Every CTA of the grid is
    // resident (grid <= occupancy x SMs), so the slowest CTA never waits.
    unsigned long long* lock;
    unsigned long long lock_base;
    int lock_blk, lock_slack;
    // unit order: 0 = z-chunk-major; G > 0 = groups of G tiles (the grid size), z chunk inside
    // the group, so a tile's next z chunk is drawn one wave after its previous one and
    // re-reads that chunk's last 2H planes from L2 (with lockstep) instead of DRAM
    int ugroup;
    // tile order inside a z-chunk row: 0 = row-major (x fastest); W > 0 = column strips of W
    // tiles, y fastest inside a strip, so y-neighbour tiles are W draws apart instead of a whole
    // tile row (units drawn close together start close together and share L2 halo rows)
    int ustrip;
    // Multi-process z-slabs (IPC halo push): boundary chunk rows first. The zb_lo bottom and zb_hi
    // top z-chunk rows of the slab (the units that read the neighbours' pushed halo planes or push
    // planes into the neighbours' halos) are drawn before the interior rows, and when the last of
    // those bflag_n units has finished, its CTA writes bflag_val into the neighbours' pass flags
    // (peer memory, system-scope release after every pushing CTA's fence). A neighbour's next
    // pass then waits only for this pass's boundary units; the interior units overlap it.
    int zb_lo, zb_hi;
    int bflag_n;           // boundary units (the first bflag_n units of the pass); 0 = off
    int* bdone;            // finished boundary units, cumulative over a step from bdone_base
    int bdone_base;
    int* bflag_dn;         // neighbour flag entries to write (peer memory) or null
    int* bflag_up;
    int bflag_val;
};

// Pass chaining. One launch may run a sequence of passes over the same tile grid. Units are
// numbered pass-major (U = q * units + u) and drawn in that order; a unit of pass q > 0 starts
// once every unit that wrote a plane it reads, or reads a plane it overwrites, has finished
// pass q-1 (chain_deps_ready). This is the device counterpart of the reference's
// dependency-counting TileScheduler (proj/src/scheduler.cpp:18-102): no grid-wide barrier and
// no kernel boundary between passes, so no per-pass ramp-up and tail. Deadlock-free because
// every dependency points at a unit drawn earlier and every drawn unit belongs to a resident
// CTA (persistent grid of at most occupancy x SMs CTAs).
constexpr int CHAIN_DESC = 6;   // distinct per-pass buffer sets in one launch
constexpr int CHAIN_MAX = 128;  // passes in one launch

struct PassDesc {               // what changes from pass to pass
    CUtensorMap vmap;           // level-0 source buffer (3-D)
    CUtensorMap umap;           // const25pt: level t0-1 (3-D)
    CUtensorMap omap;           // output: interior of dst_final (cluster: its outer CTAs)
    CUtensorMap omap_in;        // cluster kernels: output map of the inner CTAs (taller box)
    double* dst_final;          // level t0+TB (odd-nx last column stored directly)
    double* dst_penult;         // level t0+TB-1 or nullptr
    int parity0;                // parity of t0
};

struct ChainDescs {
    PassDesc d[CHAIN_DESC];         // single-pass launches use d[0] only
    unsigned char pidx[CHAIN_MAX];  // pass q uses d[pidx[q]]
    int npass;
    int* done;                      // tiles finished per (pass, z chunk), zeroed per launch
};



__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef GIRIH_MBAR_HINT
#define GIRIH_MBAR_HINT 0  // A/B: suspend-time hint (ns) of the TMA waits (0 = the default limit)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if GIRIH_MBAR_HINT > 0
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(uint32_t(GIRIH_MBAR_HINT))
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}

// the same on a precomputed shared-window address (no generic-to-shared conversion per wait)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar_s),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_plane(void* dst, const CUtensorMap* map, int x, int y,
                                               int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            int w, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}

// bulk tensor store smem -> global (async proxy) and its bulk-group bookkeeping
__device__ __forceinline__ void tma_store_plane(const CUtensorMap* map, const void* src, int x, int y,
                                                int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_but1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// thread-block clusters (y-neighbour CTAs share the halo rows of the fused levels through
// distributed shared memory)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
#ifndef GIRIH_CLUSTER_NOSYNC
#define GIRIH_CLUSTER_NOSYNC 0  // timing experiment only: no per-iteration cluster barrier
#endif
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_d2(uint32_t addr, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y)
                 : "memory");
}
// arrive on an mbarrier in another CTA of the cluster (pacing: PACE clusters)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_s32(uint32_t addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned sm_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// stores the cells of a pair selected by m (bit 0: x at a0, bit 1: y at a1; 3: both as one
// 16-byte store at a0) as predicated stores in straight-line code: the fused inner-columns-only
// tile has a half-output pair in the first and last lane of every warp, and a branchy version
// made every warp run both the vector and the scalar path
__device__ __forceinline__ void st_pair_masked(double* a0, double* a1, double2 v, uint32_t m) {
    asm volatile(
        "{\n"
        ".reg .pred p1, p2, p3;\n"
        "setp.eq.u32 p3, %4, 3;\n"
        "setp.eq.u32 p1, %4, 1;\n"
        "setp.eq.u32 p2, %4, 2;\n"
        "@p3 st.global.v2.f64 [%0], {%2, %3};\n"
        "@p1 st.global.f64 [%0], %2;\n"
        "@p2 st.global.f64 [%1], %3;\n"
        "}\n" ::"l"(a0),
        "l"(a1), "d"(v.x), "d"(v.y), "r"(m)
        : "memory");
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Work-unit geometry: unit u -> (tile x, tile y, z chunk); a unit's level-0 stream covers
// planes [za - H, zb + H).
struct UnitGeom {
    int tx, ty, za, zb;
};

__device__ __forceinline__ UnitGeom unit_geom(const PassParams& p, int u) {
    UnitGeom g;
    int zc;
    if (GIRIH_UORDER && p.ugroup > 0) {  // groups of ugroup tiles, z chunk inside the group (the last is short)
        const int txy = p.tiles_x * p.tiles_y, per = p.ugroup * p.nzc;
        const int grp = u / per, w = u - grp * per;
        const int gsz = min(p.ugroup, txy - grp * p.ugroup);
        zc = w / gsz;
        const int tile = grp * p.ugroup + (w - zc * gsz);
        g.tx = tile % p.tiles_x;
        g.ty = tile / p.tiles_x;
    } else {
        const int txy = p.tiles_x * p.tiles_y;
        zc = u / txy;
        const int tile = u - zc * txy;
        if (GIRIH_UORDER && p.ustrip > 0) {
            const int sw = p.ustrip * p.tiles_y;  // tiles per full strip
            const int strip = tile / sw, w = min(p.ustrip, p.tiles_x - strip * p.ustrip);
            const int r = tile - strip * sw;
            g.ty = r / w;
            g.tx = strip * p.ustrip + (r - g.ty * w);
        } else {
            g.ty = tile / p.tiles_x;
            g.tx = tile - g.ty * p.tiles_x;
        }
        if (p.zb_lo + p.zb_hi > 0) {  // boundary rows first: bottom rows, top rows, interior
            if (zc >= p.zb_lo) zc = zc < p.zb_lo + p.zb_hi ? p.nzc - p.zb_hi + (zc - p.zb_lo)
                                                           : zc - p.zb_hi;
        }
    }
    g.za = p.zout_lo + zc * p.zc_len;
    g.zb = min(g.za + p.zc_len, p.zout_hi);
    return g;
}

// Work distribution. Units are ordered z-chunk-major (all tiles of chunk 0, then chunk 1, ...)
// and handed out dynamically: CTA b starts with unit b, then takes gridDim.x + atomicAdd(work).
// All tiles in flight therefore sit within about one chunk of each other in z, so the halo rows
// a tile shares with its neighbours are still in L2 when the neighbour reads them (a static
// round robin lets CTAs on more crowded SMs drift ~100 planes behind, and every halo row then
// comes from DRAM a second time). The V producer (thread 0) is the only thread that draws units;
// it publishes them in a small smem queue that the aux producer and the consumers replay.
constexpr int UQ = 8;  // unit queue depth (the producer runs at most a few units ahead)

struct Cursor {
    int seq;   // this CTA's unit sequence number
    int u;     // unit id (>= total: exhausted); chained: q * units + ul
    int q;     // pass of the unit within a chained launch (0 otherwise)
    int it, n_it;
    UnitGeom ug;
};

// u: chained unit id q * units + ul (total = npass * units; single-pass launches: q = 0)
template <int H, bool CHAIN>
__device__ __forceinline__ void cursor_set(Cursor& c, const PassParams& p, int total, int seq,
                                           int u) {
    c.seq = seq;
    c.u = u;
    c.it = 0;
    c.n_it = 0;
    c.q = 0;
    if (u < total) {
        if (CHAIN) c.q = u / p.units;
        // single passes may run a sub-range [unit0, unit0 + unit_n) of the pass's units
        // (girih_gpu_update_units, the reference's update_tile)
        c.ug = unit_geom(p, CHAIN ? u - c.q * p.units : u + p.unit0);
        c.n_it = (c.ug.zb - c.ug.za) + 2 * H;
    }
}

// advance within / across units; the drawing cursor (V producer) fetches new unit ids.
// Clusters (CY > 1): the CTAs of a cluster work on the same unit (tile column, z chunk); only
// the leader CTA's producer draws, and it publishes every id into all the cluster's unit queues
// a whole unit before anyone needs it (the cluster barrier of every iteration orders the remote
// stores before the reads).
template <int H, bool CHAIN, bool DRAW, int CY = 1>
__device__ __forceinline__ void cursor_next(Cursor& c, const PassParams& p, int total,
                                            volatile int* uq, int* drawn) {
    if (++c.it >= c.n_it) {
        int next;
        if (DRAW && CY > 1) {
            next = uq[(c.seq + 1) % UQ];  // published when this cursor entered unit seq
            if (next < total) {
                const int d = int(gridDim.x) / CY + atomicAdd(p.work, 1) - p.work_base;
                const int v = d < total ? d : total;
                const uint32_t a = smem_u32(const_cast<int*>(&uq[(c.seq + 2) % UQ]));
#pragma unroll
                for (int r = 0; r < CY; ++r) st_cluster_s32(mapa_rank(a, r), v);
            }
        } else if (DRAW) {
            // the id drawn at the start of this unit; draw the one after it now, so the atomic's
            // latency hides behind a whole unit instead of stalling the producer warp
            next = *drawn;
            if (next < total) {
                // single-pass launches hand CTA b unit b first, so draws start at gridDim.x;
                // chained ones draw every unit (a CTA that is not resident yet holds none)
                const int d = (CHAIN ? 0 : int(gridDim.x)) + atomicAdd(p.work, 1) - p.work_base;
                *drawn = d < total ? d : total;
            }
            uq[(c.seq + 1) % UQ] = next;
        } else {
            next = uq[(c.seq + 1) % UQ];
        }
        cursor_set<H, CHAIN>(c, p, total, c.seq + 1, next);
    }
}

// Pass chaining: done[q * nzc + zc] counts the tiles that finished chunk zc of pass q. Unit
// (tile, zc) of pass q may start once chunk rows zc-1 .. zc+1 of pass q-1 are complete: they
// hold every unit that wrote a plane it reads or reads a plane it overwrites (the halo H is at
// most one chunk). Whole rows rather than the 3 x 3 tile neighbourhood: 3 polls instead of
// 27, and units are drawn z-chunk-major, so a row is long finished when the next pass
// reaches it.
__device__ __forceinline__ bool chain_deps_ready(const PassParams& p, const int* done, int q,
                                                 int ul) {
    const int txy = p.tiles_x * p.tiles_y;
    const int zc = ul / txy;
    const int* row = done + (q - 1) * p.nzc;
    int a, b, c;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(a) : "l"(row + max(zc - 1, 0)));
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(b) : "l"(row + zc));
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(c) : "l"(row + min(zc + 1, p.nzc - 1)));
#ifdef GIRIH_CHAIN_NODEPS
    return true;  // timing experiment only: no ordering between passes (results are wrong)
#endif
    return min(a, min(b, c)) >= txy;
}

// makes a finished unit visible (TMA stores complete, direct stores ordered by the CTA
// barrier) before its row count; the reader fences after observing the count
__device__ __forceinline__ void chain_publish(const PassParams& p, int* done, int u) {
    const int q = u / p.units, ul = u - q * p.units;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    // release: the CTA's earlier writes (ordered before this thread by the CTA barrier and,
    // for the TMA stores, by the completed bulk groups and the proxy fence) happen-before it
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(
                     done + q * p.nzc + ul / (p.tiles_x * p.tiles_y))
                 : "memory");
}
__device__ __forceinline__ void chain_acquire() {
    // pairs with the release above through the relaxed reads of the counters
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}


template <int KIND> struct STACK_OK { static constexpr bool value = true; };

// calls f(integral_constant<I>), f(integral_constant<I+1>), ... while f returns true
template <int I, int N, class F>
__device__ __forceinline__ void unroll_phases(F& f) {
    if constexpr (I < N) {
        if (f(std::integral_constant<int, I>{})) unroll_phases<I + 1, N>(f);
    }
}

template <int KIND> struct AuxArrays { static constexpr int N = KindTraits<KIND>::NC; };
template <> struct AuxArrays<K_CONST25> { static constexpr int N = 2; };  // C and level t0-1

constexpr int round16(int n) { return (n + 15) / 16 * 16; }

// CF = cluster rows CY (bits 0-7) | flags << 8. Flag 1: DOUT, the output level is stored from
// registers straight to global memory (coalesced pair stores) instead of an smem staging plane
// and a TMA store, which frees the staging planes' shared memory for deeper prefetch.
template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB = 1, int CF = 1>
struct ZwaveConfig {
    static constexpr int CY = CF & 255;
    static constexpr bool DOUT = ((CF >> 8) & 1) != 0;
    static constexpr int R = KindTraits<KIND>::R;
    // NARROW (flag 4): the threads cover only the LXC = LX - 2 XO inner columns of the box
    // instead of all LX (whose XO edge columns only ever feed neighbours). Single-step kernels:
    // a 64-column warp row is all output, so tiles of 64 columns divide the BASELINE grids
    // exactly (256 = 4 x 64, 512 = 8 x 64) where 60- and 56-column tiles leave a mostly empty
    // last tile column (256^3 const7pt: 5 x 64 computed columns per row became 4 x 64); XO is
    // the x halo the host then uses (R = 1: H + 1 = 2 keeps the TMA box origins 16-byte
    // aligned). Fused kernels: level 1 is valid on all LXC columns and the output tile is
    // LXC - 2 (TB-1) R wide (var7pt TB = 2: 62 columns from a 68-column box instead of 60 from
    // 64; the x halo XO + (TB-1) R = 3 is odd, so the tile grid starts one column into the ghost
    // cells, PassParams::xorg).
    static constexpr bool NARROW = ((CF >> 10) & 1) != 0;
    static constexpr int XO = NARROW ? 2 * ((R + 1) / 2) : 0;
    static constexpr int LXC = LX - 2 * XO;  // columns the threads compute
    static constexpr int Q = 2 * R + 1;     // z window of one level
    // z neighbours come from per-thread register queues; smem only holds the centre planes
    // that other threads read for x/y neighbours: R+1 planes per computed level (written R
    // iterations before they are read) and R+1+P for the TMA-fed level 0
    static constexpr int QL = R + 1;        // level-s (s >= 1) centre-plane ring depth
    static constexpr int NR0 = R + 1 + P;   // level-0 TMA ring depth
    static constexpr int H = TB * R;        // halo of the loaded tile
    static constexpr int OY = LY - 2 * H;   // output tile height (x: runtime, halo H or H+1)
    // Thread-block clusters of CY CTAs stacked along y (CY > 1, TB >= 2). CTA c's box starts
    // c*OWN rows above CTA c-1's, so neighbouring boxes overlap by the 2R level-0 rows each
    // needs from the other. Every CTA computes its OWN rows [R, LY-R) at every level; the rows
    // of level s-1 beyond an INNER edge are the neighbour's own rows, which it pushes into this
    // CTA's ring through distributed shared memory. Only the cluster's outer edges keep the
    // trapezoid halo, so the redundant rows per CTA drop from 2(TB-1)R to 2(TB-1)R/CY.
    // PACE (flag 2): the cluster only paces its CTAs. Each CTA computes an ordinary trapezoid
    // tile (OY output rows, the box of CTA c starts c*OY rows above CTA c-1's) and nothing is
    // exchanged; the per-iteration cluster barrier keeps the CY y-neighbours on the same z
    // plane, so the level-0 and coefficient rows their boxes share are read from DRAM once and
    // hit L2 for the second reader (free-running CTAs drift apart by more than a plane's L2
    // lifetime).
    static constexpr bool PACE = ((CF >> 9) & 1) != 0;
    static constexpr bool SHARE = CY > 1 && !PACE;                // DSMEM-shared halo rows
    static constexpr int OWN = PACE ? OY : LY - 2 * R;
    static constexpr int OYS = SHARE ? OWN : OY;                  // widest output rows of a CTA
    static constexpr int OYC = CY > 1 ? (PACE ? CY * OY : CY * OWN - 2 * (TB - 1) * R) : OY;
    static constexpr int OYE = SHARE ? LY - R - H : OY;           // outer CTAs' output rows
    static constexpr int OXM = NARROW ? LXC - 2 * (TB - 1) * R : LX - 2 * H;  // widest output tile
    static constexpr int CELLS = LX * LY;
    static constexpr int CELLS_S = round16(CELLS);  // ring slot stride (TMA: 128-byte aligned)
    // threads cover the level-1 valid rows [R, LY - R) only: the R outermost rows of the
    // loaded box are neighbours, never computed (for TB = 1 that is exactly the output rows)
    static constexpr int CR = LY - 2 * R;
    static constexpr int PPT = CR * LXC / (2 * NT);  // x-pairs of cells per thread
    // STACK (64-wide tiles, >= 2 pairs per thread): a warp owns whole rows and a thread the
    // same pair column in PPT consecutive rows, so the y neighbours of its pairs are one column
    // window of PPT+2R pair loads instead of 2R loads per pair (radius 4: 46% fewer LDS.128)
    static constexpr bool STACK = LXC == 64 && PPT >= 2 && STACK_OK<KIND>::value;
    static constexpr int XA = 2 * ((R + 1) / 2);  // pair-aligned x reach (R=1: 2, R=4: 4)
    static constexpr int NRING = NR0 + (TB - 1) * QL;
    // aux (coefficient) planes: the level-1 area, x origin kept 16-byte aligned
    static constexpr int NAUX = AuxArrays<KIND>::N;
    static constexpr int AXO = NARROW ? XO : R & ~1, AYO = R;
    static constexpr int AX = LX - 2 * AXO, AY = LY - 2 * AYO;
    static constexpr int AYX = AX * AY;
    // var7pt with TB = 2 keeps each pair's coefficients in registers from level 1 to level 2
    // (same cells, R iterations later), so only level 1 reads the aux ring (deeper TB would need
    // 28 more registers per level and spills)
    static constexpr bool CQ = KIND == K_VAR7 && TB == 2;
    static constexpr int NAR = NAUX > 0 ? (CQ ? 1 : (TB - 1) * R + 1) + PA : 0;  // aux ring depth
    static constexpr int AUXPLANE = NAUX * AYX;
    // guard rows before/after the rings: unconditional edge-cell stencils stay in bounds
    static constexpr int GUARD = NARROW ? 16 : round16(LX * R + R + 8);  // (NARROW stays in the box)
    static constexpr int STAGE = DOUT ? 0 : round16(OXM * OYS);  // one output staging plane
    static constexpr size_t SMEM_DOUBLES = size_t(GUARD) * 2 + size_t(NRING) * CELLS_S +
                                           size_t(NAR) * AUXPLANE + 3 * size_t(STAGE);
    static constexpr size_t SMEM = SMEM_DOUBLES * sizeof(double) + (NR0 + NAR) * sizeof(uint64_t);
    static_assert((CR * LXC) % (2 * NT) == 0, "computed rows must split evenly into cell pairs");
    static_assert(!NARROW || (CY == 1 && (TB == 1 || DOUT)), "NARROW: non-cluster kernels; fused ones store directly");
    static_assert(NT % 32 == 0, "whole warps");
    static_assert(!STACK || CR % (NT / 32) == 0, "STACK: every warp owns whole rows");
    static_assert(LXC % 32 == 0, "a warp must cover one tile row (warp-uniform row activity)");
    static_assert(LX - 2 * H - 2 > 0 && OYE > 0, "tile too small for the halo (x halo may be H+1)");
    static_assert(LX <= 256 && LY <= 256, "TMA box limit");
    static_assert((LX * 8) % 16 == 0 && (AX * 8) % 16 == 0, "TMA inner box must be 16-byte multiple");
    static_assert((CELLS_S * 8) % 128 == 0 && (AYX * 8) % 128 == 0, "TMA smem boxes 128-byte aligned");
    static_assert(SMEM <= 232448, "exceeds 227 KB of shared memory per CTA");
    static_assert(CY == 1 || PACE || (TB >= 2 && OYE > 0 && OWN >= 2 * R && CY <= 16),
                  "clusters share fused-level halo rows: TB >= 2, outer CTAs need output rows");
};

// CHAIN = false: one pass (descriptors d[0]); true: cd.npass chained passes. The two are
// separate instantiations so that single-pass launches carry none of the chaining state (the
// 128-register var7pt CTA spills otherwise, and shared-memory producer state cost 30%).
template <int KIND, int TB, int LX, int LY, int NT, int P, int PA, int MINB, bool CHAIN, int CF = 1,
          bool INSTR = false>
__global__ void __launch_bounds__(NT, (CHAIN && GIRIH_CHAIN_MINB_DROP && MINB > 1) ? MINB - 1 : MINB)
    zwave_kernel(const __grid_constant__ CUtensorMap cmap,  // coefficient block (4-D)
                 const __grid_constant__ ChainDescs cd,     // per-pass buffers and maps
                 const __grid_constant__ PassParams p) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P, PA, MINB, CF>;
    constexpr int CY = CFG::CY;
    constexpr bool DOUT = CFG::DOUT;
    static_assert(CY == 1 || !CHAIN, "cluster kernels run single passes");
    static_assert(!INSTR || !CHAIN, "instrumented kernels run single passes");
    constexpr int R = CFG::R, QL = CFG::QL, NR0 = CFG::NR0, H = CFG::H;
    constexpr int CELLS = CFG::CELLS, CELLS_S = CFG::CELLS_S, PPT = CFG::PPT, XA = CFG::XA;
    constexpr bool NARROW = CFG::NARROW;
    constexpr int XO = CFG::XO, LXC = CFG::LXC;
    constexpr int OWN = CFG::OWN, OYC = CFG::OYC;
    constexpr int NAUX = CFG::NAUX, NAR = CFG::NAR, AXO = CFG::AXO, AYO = CFG::AYO;
    constexpr bool CQ = CFG::CQ;
    // PACE clusters: no per-plane cluster barrier. Thread 0 of each CTA arrives, per finished
    // iteration, on its y-neighbours' pace barriers (a ring of PK mbarriers, one per iteration
    // mod PK) and, before issuing the next loads, waits until the neighbours have finished all
    // but the last PD iterations it has: the neighbours stay within PD planes of each other
    // with no stall while they are (a neighbour is never more than PD+1 iterations ahead, so
    // PK > 2(PD+1) keeps the ring's phases unambiguous).
    constexpr bool PACE = CFG::PACE;
    constexpr bool CSYNC = CY > 1 && !PACE && !GIRIH_CLUSTER_NOSYNC;  // per-plane cluster barrier
    constexpr int PK = 8, PD = GIRIH_PACE_LAG;
    static_assert(PK > 2 * (PD + 1), "pace ring too short for the lag");
    // x neighbours by warp shuffle (misaligned pair loads cost two shared-memory wavefronts
    // per quarter warp). Measured (same box): const7pt single-pass +4.5% (512^3); const7pt
    // chained -15%, var7pt -2%, const25pt -5% (radius 4: 16 shuffles per pair), var25pt +-0.
    constexpr bool XSHFL = GIRIH_XSHFL && KIND == K_CONST7 && !CHAIN;
    constexpr int AX = CFG::AX, AYX = CFG::AYX, AUXPLANE = CFG::AUXPLANE;
    constexpr int GUARD = CFG::GUARD, STAGE = CFG::STAGE;
    constexpr uint32_t PLANE_BYTES = CELLS * sizeof(double);
    constexpr uint32_t AUX_BYTES = AUXPLANE * sizeof(double);
    constexpr int KOFF = QL * 4096;  // keeps ring indices of planes below 0 non-negative
    // stream counters start at a common multiple of the ring depths (first phase parity 0)
    constexpr uint32_t G0 = 8u * NR0 * (NAR > 0 ? NAR : 1);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring0 = reinterpret_cast<double*>(smem_raw) + GUARD;
    double* ringL = ring0 + NR0 * CELLS_S;           // level s (1..TB-1): ringL + (s-1)*QL*CELLS
    double* auxr = ringL + (TB - 1) * QL * CELLS_S;  // aux planes: NAR x [NAUX][AY][AX]
    double* stage = auxr + NAR * AUXPLANE + GUARD; // 3 output staging planes [OYS][ox]
    uint64_t* vbar = reinterpret_cast<uint64_t*>(stage + 3 * STAGE);
    uint64_t* abar = vbar + NR0;

    const int tid = threadIdx.x;
    __shared__ uint64_t pbar[PACE ? PK : 1];
    // cluster position (CY > 1): rank c owns box rows [R, LY-R) of the cluster tile's c-th box;
    // the outer CTAs (c = 0, CY-1) keep the trapezoid halo on their outer side
    const int crank = CY > 1 ? int(cluster_ctarank()) : 0;
    // (PACE: every CTA is a whole trapezoid tile, both edges outer)
    const bool lo_edge = CFG::PACE || crank == 0, hi_edge = CFG::PACE || crank == CY - 1;
    const int oy_lo = lo_edge ? H : R;  // first output row of this CTA's box
    if (tid == 0) {
        for (int b = 0; b < NR0; ++b) mbar_init(&vbar[b], 1);
        for (int b = 0; b < NAR; ++b) mbar_init(&abar[b], 1);
        if constexpr (PACE)  // one arrival per y-neighbour and iteration
            for (int b = 0; b < PK; ++b)
                mbar_init(&pbar[b], uint32_t((crank > 0 ? 1 : 0) + (crank < CY - 1 ? 1 : 0)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();

    // PACE: iteration i finished -> one arrival on each y-neighbour's pace barrier i % PK
    [[maybe_unused]] auto pace_arrive = [&](uint32_t i) {
        const uint32_t a = smem_u32(&pbar[PACE ? i % PK : 0]);
        if (crank > 0) mbar_arrive_remote(mapa_rank(a, uint32_t(crank - 1)));
        if (crank < CY - 1) mbar_arrive_remote(mapa_rank(a, uint32_t(crank + 1)));
    };
    // ---- producers (thread 0): V runs P elements ahead, aux PA elements ahead ----
    __shared__ int uq[UQ];
    const int total = CHAIN ? cd.npass * p.units : p.unit_n;  // units of the launch
    Cursor vcur{}, acur{};
    uint32_t vnext = G0, anext = G0;
    int drawn = 0;  // producer: next unit id, drawn one unit ahead
    bool lock_done = false;  // lockstep: this CTA has released the others
    // chained launches: the V cursor's unit passed its dependency check; the store thread's
    // finished unit whose last plane is the pending store
    bool vready = false;
    int pub_next = -1;
    // returns false when a chained unit's dependencies are not met yet and `must` is false
    auto issue_v = [&](bool must) -> bool {
        if (vcur.u >= total) {
            if constexpr (!CHAIN && CY == 1 && GIRIH_LOCK) {
                if (p.lock && !lock_done) {  // out of units: release the others for good
                    const unsigned arrived = (vnext - G0 + unsigned(p.lock_blk) - 1) / unsigned(p.lock_blk);
                    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p.lock),
                                 "l"((1ull << 32) - arrived)
                                 : "memory");
                    lock_done = true;
                }
            }
            return false;
        }
        if constexpr (!CHAIN && CY == 1 && GIRIH_LOCK) {
            if (p.lock && (vnext - G0) % unsigned(p.lock_blk) == 0) {
                const unsigned m = (vnext - G0) / unsigned(p.lock_blk);  // block of this plane
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(p.lock) : "memory");
                if (m >= unsigned(p.lock_slack)) {
                    const unsigned long long need =
                        p.lock_base + (unsigned long long)(m - p.lock_slack + 1) * gridDim.x;
                    long long spins = 0;
                    for (;;) {
                        unsigned long long a;
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p.lock));
                        if (a >= need) break;
                        __nanosleep(32);
                        if (++spins > (1ll << 28)) {  // watchdog: flag for the host, proceed
                            atomicExch(p.work + 1, 1);
                            break;
                        }
                    }
                }
            }
        }
        if constexpr (CHAIN) {
            if (vcur.it == 0 && vcur.q > 0 && !vready) {
                const int ul = vcur.u - vcur.q * p.units;
                if (!chain_deps_ready(p, cd.done, vcur.q, ul)) {
                    if (!must) return false;  // retry next iteration
                    // the consumer needs this plane now. If this CTA's own last unit is a
                    // dependency, the store thread publishes it at the top of this same
                    // iteration (before the barrier this thread is held at), so the wait ends.
                    // watchdog (~2 minutes): a wait that long is a bug; flag it for the host
                    // (girih_gpu_step then fails with GIRIH_ECUDA) and proceed rather than hang
                    // the GPU or kill the context with a trap
                    long long spins = 0;
                    while (!chain_deps_ready(p, cd.done, vcur.q, ul)) {
                        __nanosleep(128);
                        if (++spins > (1ll << 30)) {
                            atomicExch(p.work + 1, 1);
                            break;
                        }
                    }
                }
                chain_acquire();
                vready = true;
            }
        }
        const int j = vcur.ug.za - H + vcur.it;
        const int slot = int(vnext % NR0);
        const int xd = p.off + vcur.ug.tx * p.ox + p.xorg;  // even by construction
        const int yd = vcur.ug.ty * OYC + crank * OWN + R - H;
        mbar_arrive_expect_tx(&vbar[slot], PLANE_BYTES);
        tma_load_plane(ring0 + slot * CELLS_S, &cd.d[CHAIN ? cd.pidx[vcur.q] : 0].vmap, xd, yd, j,
                       &vbar[slot]);
        ++vnext;
        if (CY > 1 && crank > 0)  // cluster members replay the leader's units
            cursor_next<H, CHAIN, false>(vcur, p, total, uq, nullptr);
        else
            cursor_next<H, CHAIN, true, CY>(vcur, p, total, uq, &drawn);
        if (CHAIN && vcur.it == 0) vready = false;
        return true;
    };
    auto issue_a = [&]() {
        if constexpr (NAUX > 0) {
            if (acur.u >= total) return;
            const int k1 = acur.ug.za - H + acur.it - R;  // level-1 plane of that iteration
            const int slot = int(anext % NAR);
            const int xd = p.off + acur.ug.tx * p.ox + p.xorg + AXO;
            const int yd = acur.ug.ty * OYC + crank * OWN + R - H + AYO;
            if (acur.it < 2 * R) {
                // no level reads the aux plane of the first 2R iterations of a unit: complete
                // the phase without moving data
                mbar_arrive(&abar[slot]);
                ++anext;
                cursor_next<H, CHAIN, false>(acur, p, total, uq, nullptr);
                return;
            }
            mbar_arrive_expect_tx(&abar[slot], AUX_BYTES);
            double* dst = auxr + slot * AUXPLANE;
            if constexpr (KIND == K_CONST25) {
                tma_load_plane(dst, &cmap, xd, yd, k1, &abar[slot]);
                tma_load_plane(dst + AYX, &cd.d[CHAIN ? cd.pidx[acur.q] : 0].umap, xd, yd, k1,
                               &abar[slot]);
            } else {
                tma_load_4d(dst, &cmap, xd, yd, k1, 0, &abar[slot]);
            }
            ++anext;
            cursor_next<H, CHAIN, false>(acur, p, total, uq, nullptr);
        }
    };
    static_assert(P >= PA, "the V producer draws units and must lead the aux producer");
    if constexpr (CY > 1) {
        // the leader hands out the cluster's first two units (cluster c starts with unit c),
        // once every CTA of the cluster is running (distributed shared memory is only valid then)
        cluster_arrive();
        cluster_wait();
        if (tid == 0 && crank == 0) {
            const int ncl = int(gridDim.x) / CY, cid = int(blockIdx.x) / CY;
            const int u0 = cid < total ? cid : total;
            int u1 = total;
            if (u0 < total) {
                const int d = ncl + atomicAdd(p.work, 1) - p.work_base;
                u1 = d < total ? d : total;
            }
#pragma unroll
            for (int r = 0; r < CY; ++r) {
                st_cluster_s32(mapa_rank(smem_u32(&uq[0]), r), u0);
                st_cluster_s32(mapa_rank(smem_u32(&uq[1]), r), u1);
            }
        }
        cluster_arrive();  // the queues (and every CTA's mbarriers) are initialised
        cluster_wait();
        if (tid == 0) {
            const int u0 = reinterpret_cast<volatile int*>(uq)[0];
            cursor_set<H, CHAIN>(vcur, p, total, 0, u0);
            cursor_set<H, CHAIN>(acur, p, total, 0, u0);
            for (int e = 0; e < P; ++e) issue_v(true);
            for (int e = 0; e < PA; ++e) issue_a();
        }
        if constexpr (!PACE) cluster_arrive();  // pairs with the first iteration's wait
    } else if (tid == 0) {
        // single-pass launches: the first unit is blockIdx.x. Chained launches draw it too, so
        // that every unit another CTA may wait for belongs to a CTA that is already running
        // (drawing takes residency; launch order alone would not guarantee it).
        int u0;
        if constexpr (CHAIN) {
            const int d0 = atomicAdd(p.work, 1) - p.work_base;
            u0 = d0 < total ? d0 : total;
        } else {
            u0 = blockIdx.x < total ? int(blockIdx.x) : total;
        }
        uq[0] = u0;
        if (u0 < total) {
            const int d = (CHAIN ? 0 : int(gridDim.x)) + atomicAdd(p.work, 1) - p.work_base;
            drawn = d < total ? d : total;
        } else {
            drawn = total;
        }
        cursor_set<H, CHAIN>(vcur, p, total, 0, u0);
        cursor_set<H, CHAIN>(acur, p, total, 0, u0);
        if constexpr (!CHAIN) {  // chained launches issue from the first iteration on
            for (int e = 0; e < P; ++e) issue_v(true);
            for (int e = 0; e < PA; ++e) issue_a();
        }
    }
    // output store pending from the previous iteration. In CTAs of 2-8 warps (latency-bound:
    // const7pt +4%, const25pt +3%) the output stores and their bulk-group waits run on warp 1
    // (bulk groups are per thread), off the load producer's (thread 0's) per-plane critical
    // path; the 14-warp var7pt TB=2 CTA keeps them on thread 0 (-2% otherwise). In chained
    // launches the store thread also publishes finished units (bulk groups are per thread).
    constexpr int STORE_TID = (NT >= 64 && NT <= 256) ? 32 : 0;
    bool pend = false, stored_now = false;
    int pend_x = 0, pend_y = 0, pend_z = 0, pend_b = 0, pend_q = 0;

    // ---- per-thread constants. A thread owns x-PAIRS of cells (2 consecutive x): every
    //      neighbour access is a 16-byte LDS.128 and the x neighbourhood of a pair comes from
    //      XA+1 aligned pair loads. Bit 2i+q of a mask = cell q of pair i. ----
    int lcell[PPT], dyv[PPT], ai[PPT], sidx[PPT];
    uint32_t out_mask = 0;
    // box row / column of pair i's first cell, straight from the thread index (NARROW boxes
    // are 68 or 72 columns wide: no division by LX in the per-unit mask setup)
    auto cell_ly = [&](int i) -> int {
        return CFG::STACK ? R + (tid >> 5) * PPT + i
               : NARROW   ? R + 2 * (tid + NT * i) / LXC
                          : (2 * (tid + NT * i) + R * LX) / LX;
    };
    auto cell_lx = [&](int i) -> int {
        return CFG::STACK ? XO + 2 * (tid & 31)
               : NARROW   ? XO + 2 * (tid + NT * i) % LXC
                          : (2 * (tid + NT * i) + R * LX) % LX;
    };
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
        // first cell of the pair (even)
        const int c = CFG::STACK ? (R + (tid >> 5) * PPT + i) * LX + XO + 2 * (tid & 31)
                      : NARROW   ? (R + 2 * (tid + NT * i) / LXC) * LX + XO + 2 * (tid + NT * i) % LXC
                                 : 2 * (tid + NT * i) + R * LX;
        lcell[i] = c;
        const int lx = cell_lx(i), ly = cell_ly(i);
        // distance to the nearest box edge that has a trapezoid halo (inner cluster edges have
        // none: the neighbour supplies the rows beyond them)
        const int dy = min((CY > 1 && !lo_edge) ? 1 << 20 : ly,
                           (CY > 1 && !hi_edge) ? 1 << 20 : LY - 1 - ly);
        dyv[i] = dy;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int dx = min(lx + q, LX - 1 - lx - q);
            if (dx >= p.hx && dy >= H) out_mask |= 1u << (2 * i + q);
        }
        ai[i] = (ly - AYO) * AX + (lx - AXO);
        sidx[i] = (ly - oy_lo) * p.ox + (lx - p.hx);
    }
    // pairs whose whole warp lies outside the level-s valid rows skip the stencil (warp-uniform;
    // their values are never read): bit (s-1)*PPT + i. Only for R = 1: the 25-point bodies are
    // long enough that the per-pair branch costs more interleaving than the skipped work saves.
    static_assert(TB * PPT <= 32, "warp skip mask");
    uint32_t wskip = 0;
#pragma unroll
    for (int s = 1; s <= (R == 1 ? TB : 0); ++s)
#pragma unroll
        for (int i = 0; i < PPT; ++i)
            if (__all_sync(0xffffffffu, dyv[i] < s * R)) wskip |= 1u << ((s - 1) * PPT + i);
    // a chained unit's pass-dependent values, read where needed (rare paths) from shared
    // memory instead of being held in registers by every thread
    struct UnitState {
        const double* ghost_s[TB + 1];  // parity-(t0+s) pristine field (ghost values of level s)
        double* dst_final;
        double* dst_penult;
    };
    // double-buffered by unit sequence: slower warps may still read the previous unit's copy
    // in its last iteration while thread 0 fills the next one (no barrier in between)
    __shared__ UnitState SU2[2];
    const bool has_penult_1 = p.dst_penult != nullptr;  // single-pass launches
    // coefficient queue (CQ): cq[L][pair] = coefficients level 1 used L+1 iterations ago
    // PHQ (single-pass var7pt TB = 2, A/B builds): the 2-entry z queues and the coefficient queue
    // rotate by renaming over 2 unrolled iteration phases (level 1 fills one of two coefficient
    // register sets, level 2 reads the other) instead of being shifted (the shifts are 44 of
    // the kernel's 282 instructions per warp and plane). Measured: the two-phase body spills
    // 48 B at the 128-register cap and runs 13% slower (122.5 K vs 141.6 K at 1024^3)
    constexpr bool PHQ = GIRIH_PHQ && CQ && TB == 2 && R == 1 && !CHAIN && CY == 1;
    constexpr int CQD = CQ ? TB - 1 : 1, CQN = CQ ? 7 : 1;
    double2 cq[CQD][PPT][CQN], cnew[PPT][CQN];
    double2 cqr[PHQ ? 2 : 1][PPT][CQN];  // PHQ: the two coefficient sets (phase parity)
    // per-thread z queues: zq[L][pair][d] = level L at plane (newest_L - 2R + d), d = 0..2R-1
    // ZPS (single-step radius-4 passes): the z+ neighbours k+1..k+R-1 are read from the level-0
    // ring, which holds planes k..k+R anyway, so the queue keeps only k-R..k-1 (fewer registers;
    // it is fed with the centre plane k instead of the newest plane). Measured (same box): the
    // chained const25pt kernel stops spilling, +14-18% at 64^3-256^3; single-pass const25pt -1%,
    // chained var25pt 128^3 -8%, so it is on for chained const25pt only.
    // PHZ (single-pass const25pt): the 4-entry z- queue rotates by renaming over 4 unrolled
    // iteration phases instead of 64 register moves per warp-iteration; it needs ZPS's short
    // queue to fit the register budget (the 8-entry version spilled)
    constexpr bool PHZ = (GIRIH_PHZ && TB == 1 &&
                          (GIRIH_PHZ_ALL ? R == 4 : (KIND == K_CONST25 && !CHAIN))) || PHQ;
    constexpr bool ZPS = GIRIH_ZPS && TB == 1 && ((KIND == K_CONST25 && (CHAIN || GIRIH_ZPS_ALL25)) || PHZ);
    constexpr int ZQD = ZPS ? R : 2 * R;
    double2 zq[TB][PPT][ZQD];
#pragma unroll
    for (int L = 0; L < TB; ++L)
#pragma unroll
        for (int i = 0; i < PPT; ++i)
#pragma unroll
            for (int d = 0; d < ZQD; ++d) zq[L][i][d] = make_double2(0.0, 0.0);

    __syncthreads();  // uq[0] visible
    uint32_t g = G0;  // consumer's global element index
    // g's ring slots and mbarrier phase parities, advanced with g instead of recomputed every
    // iteration by divisions by the ring depths (6 and 2-3 planes: not powers of two); G0 is a
    // multiple of 2 NR0 and 2 NAR, so both start at slot 0, parity 0
    int gs = 0, as = 0;
    uint32_t gph = 0, aph = 0;
    const uint32_t vbar_s = smem_u32(vbar), abar_s = smem_u32(abar);
    // slot of the plane `back` iterations before g's
    auto vslot = [&](int back) -> int {
        const int sl = gs - back % NR0;
        return sl < 0 ? sl + NR0 : sl;
    };
    auto aslot = [&](int back) -> int {
        const int sl = as - back % (NAR > 0 ? NAR : 1);
        return sl < 0 ? sl + NAR : sl;
    };
    unsigned long long unit_t0 = 0;  // instrumentation: start of thread 0's current unit
    for (int seq = 0;; ++seq) {
        const int u = reinterpret_cast<volatile int*>(uq)[seq % UQ];
        if (u >= total) break;
        const UnitGeom ug = unit_geom(p, CHAIN ? u % p.units : u + p.unit0);
        // chained: bit 0 = the unit's pass writes the penult level, bits 1.. = that pass
        int uflags = 0;
        if constexpr (CHAIN) {
            const int q = u / p.units;
            const PassDesc& pd = cd.d[cd.pidx[q]];
            uflags = (q << 1) | (pd.dst_penult != nullptr ? 1 : 0);
            if (tid == 0) {  // published by the __syncthreads_or below
                UnitState& SU = SU2[seq & 1];
#pragma unroll
                for (int s2 = 0; s2 <= TB; ++s2) SU.ghost_s[s2] = p.ghost[(pd.parity0 + s2) & 1];
                SU.dst_final = pd.dst_final;
                SU.dst_penult = pd.dst_penult;
            }
        }
        const int n_it = (ug.zb - ug.za) + 2 * H;
        const int xa0 = ug.tx * p.ox + p.xorg;  // allocated x of local lx = 0
        const int ya0 = ug.ty * OYC + crank * OWN + R - H;

        // ghost columns (ghost value instead of the stencil) and in-allocation columns
        uint32_t ghost_mask = 0, ok_mask = 0, odd_mask = 0;
        int colidx[2 * PPT];  // row offset within a plane (allocated coordinates)
#pragma unroll
        for (int i = 0; i < PPT; ++i)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int b = 2 * i + q;
                const int xa = xa0 + cell_lx(i) + q, ya = ya0 + cell_ly(i);
                if (xa >= 0 && xa < p.X && ya >= 0 && ya < p.Y) ok_mask |= 1u << b;
                if (xa < R || xa >= R + p.nx || ya < R || ya >= R + p.ny) ghost_mask |= 1u << b;
                // TMA stores clip x at 16-byte granularity, so the store map stops at an even
                // nx and an odd nx's last interior column is stored directly (odd_mask)
                if ((p.nx & 1) && xa == R + p.nx - 1 && ya >= R && ya < R + p.ny &&
                    ((out_mask >> b) & 1))
                    odd_mask |= 1u << b;
                const int cx = min(max(xa, 0), p.X - 1), cy = min(max(ya, 0), p.Y - 1);
                colidx[b] = cy * p.pitch + p.off + cx;
            }
        const uint32_t col_fix = ghost_mask & ok_mask;
        const uint32_t dmask = out_mask & ~ghost_mask;  // cells this thread stores (direct output)
        const bool any_ghost_col = __syncthreads_or(col_fix != 0);
        const bool any_odd_col = (p.nx & 1) && ug.tx == p.tiles_x - 1;  // owner of the last column

        // one z-plane iteration; PH = phase of the rotating z queue (always 0 unless PHZ)
        auto iteration = [&](auto PHc, const int it) {
            constexpr int PH = decltype(PHc)::value;
            const int j = ug.za - H + it;  // level-0 plane of this iteration
            __syncthreads();               // previous iteration's smem reads/writes are complete
#ifdef GIRIH_ZWAVE_TRACE
            const bool tr = p.ptrace && blockIdx.x == 0 && (tid == 0 || tid == 32) && g - G0 < 4096;
#else
            constexpr bool tr = false;  // build with -DGIRIH_ZWAVE_TRACE for phase clocks
#endif
            unsigned long long* trp = tr ? p.ptrace + ((g - G0) * 2 + (tid == 32)) * 4 : nullptr;
            if (tr) trp[0] = clock64();
            if (tid == STORE_TID) {
                stored_now = false;
                if (pend) {  // output plane of the previous iteration (staging fenced by writers)
                    const PassDesc& od = cd.d[CHAIN ? cd.pidx[pend_q] : 0];
                    tma_store_plane((CY > 1 && !lo_edge && !hi_edge) ? &od.omap_in : &od.omap,
                                    stage + pend_b * STAGE, pend_x, pend_y, pend_z);
                    bulk_commit();
                    pend = false;
                    stored_now = true;
                }
                if constexpr (CHAIN) {
                    // a finished unit (its last plane was just stored) is published as soon as
                    // its stores have completed: the producer may be waiting for it right now
                    if (pub_next >= 0) {
                        bulk_wait_all();
                        chain_publish(p, cd.done, pub_next);
                        pub_next = -1;
                    }
                }
            }
            if (tid == 0) {
                if constexpr (CHAIN) {
                    // V planes up to g + P (at least plane g, which the consumer waits for
                    // next), aux planes up to g + PA but never past V, which checks a unit's
                    // dependencies before its first plane
                    while (vnext <= g + P)
                        if (!issue_v(vnext <= g)) break;
                    if constexpr (NAUX > 0)
                        while (anext <= g + PA && anext < vnext) issue_a();
                } else {
                    if constexpr (PACE) {
                        const uint32_t m = g - G0;  // iterations this CTA has finished
                        if (m > 0) pace_arrive(m - 1);
                        if (m > PD) {
                            const uint32_t i = m - 1 - PD;  // neighbours must have finished it
                            // acquire at cluster scope: the leader's remote unit-queue
                            // stores before its arrivals are visible after this wait
                            mbar_wait_cluster(&pbar[i % PK], (i / PK) & 1);
                        }
                    }
                    issue_v(true);
                    issue_a();
                }
            }
            // ghost values of the intermediate levels this iteration (boundary tiles and ghost
            // planes only), loaded before the TMA waits so their latency overlaps them. Level TB
            // needs none: the interior-only store map clips its ghost cells.
            double2 gh[TB > 1 ? TB - 1 : 1][PPT];
#pragma unroll
            for (int s = 1; s < TB; ++s) {
                const int k = j - s * R;
                if (it < 2 * s * R || k < 0 || k >= p.Zloc) continue;
                const int kg = k + p.zoff;
                const bool plane_ghost = kg < R || kg >= R + p.nzg;
                if (!(plane_ghost || any_ghost_col)) continue;
                const double* ghost =
                    (CHAIN ? SU2[seq & 1].ghost_s[s] : p.ghost[(p.parity0 + s) & 1]) + (long long)k * p.plane;
                const uint32_t fix = plane_ghost ? ok_mask : col_fix;
#pragma unroll
                for (int i = 0; i < PPT; ++i) {
                    if (dyv[i] < s * R) continue;
                    if ((fix >> (2 * i)) & 1) gh[s - 1][i].x = __ldg(ghost + colidx[2 * i]);
                    if ((fix >> (2 * i + 1)) & 1) gh[s - 1][i].y = __ldg(ghost + colidx[2 * i + 1]);
                }
            }
            mbar_wait_s(vbar_s + 8u * uint32_t(gs), gph);
            if constexpr (NAUX > 0) mbar_wait_s(abar_s + 8u * uint32_t(as), aph);
            if (tr) trp[1] = clock64();

            // level-0 newest plane j into the level-0 z queue input (one LDS.128 per pair)
            double2 newest[PPT];  // level s-1 at (pair, k_s + R), produced this iteration
            {
                const double2* pj = reinterpret_cast<const double2*>(ring0 + gs * CELLS_S);
#pragma unroll
                for (int i = 0; i < PPT; ++i) newest[i] = pj[lcell[i] >> 1];
            }
            double2 ctrk[ZPS ? PPT : 1];  // ZPS: level 0 at the centre plane k = j - R
            if constexpr (ZPS) {
                const double2* pk = reinterpret_cast<const double2*>(ring0 + vslot(R) * CELLS_S);
#pragma unroll
                for (int i = 0; i < PPT; ++i) ctrk[i] = pk[lcell[i] >> 1];
            }
            // value of level L at its newest plane (j - L R) this iteration; the z queues advance
            // by one plane EVERY iteration so zq[L] always holds planes j-LR-2R .. j-LR-1 (entries
            // of planes a level did not compute are never read by a valid cell)
            double2 fresh[TB][PPT];
#pragma unroll
            for (int L = 0; L < TB; ++L)
#pragma unroll
                for (int i = 0; i < PPT; ++i)
                    fresh[L][i] = L == 0 ? (ZPS ? ctrk[ZPS ? i : 0] : newest[i]) : make_double2(0.0, 0.0);
            bool staged = false;
            int ring_slot[TB];  // centre-ring slot each level writes this iteration (-1: none)
#pragma unroll
            for (int L = 0; L < TB; ++L) ring_slot[L] = -1;
            // clusters: levels >= 2 read halo rows the neighbour CTAs pushed at the end of an
            // earlier iteration; the wait sits after level 1 so the barrier's latency hides
            // behind it (the arrive is at the end of the previous iteration)
            [[maybe_unused]] bool cwaited = false;
#pragma unroll
            for (int s = 1; s <= TB; ++s) {
                if constexpr (CSYNC) {
                    if (s == 2) {
                        cluster_wait();
                        cwaited = true;
                    }
                }
                const int k = j - s * R;  // plane of level s
                // lower bounds are monotone in s (higher levels sit on lower planes)
                if (it < 2 * s * R || k < 0) break;
                // above the buffer: skip this level only; level s+1 sits R planes lower (a
                // ghost plane there, so it never reads this level's value)
                if (k >= p.Zloc) continue;
                const int kg = k + p.zoff;
                const bool plane_ghost = kg < R || kg >= R + p.nzg;
                // centre plane k of level s-1 (x/y neighbours, other threads' values)
                const double2* pc = reinterpret_cast<const double2*>(
                    s == 1 ? ring0 + vslot(R) * CELLS_S
                           : ringL + ((s - 2) * QL + (k + KOFF) % QL) * CELLS_S);
                const double2* aux = NAUX > 0 ? reinterpret_cast<const double2*>(
                                                    auxr + aslot((s - 1) * R) * AUXPLANE)
                                              : nullptr;

                // (1) stencil for every pair of the valid rows; cells outside the valid area in x
                //     compute garbage that no valid cell ever reads (guard rows keep the smem
                //     reads in bounds)
                double2 val[PPT];
                // STACK: this thread's column window, rows r0-R .. r0+PPT-1+R
                double2 colw[CFG::STACK ? PPT + 2 * R : 1];
                if constexpr (CFG::STACK) {
                    const int hb = (lcell[0] >> 1) - R * (LX / 2);
#pragma unroll
                    for (int m = 0; m < PPT + 2 * R; ++m) colw[m] = pc[hb + m * (LX / 2)];
                }
#pragma unroll
                for (int i = 0; i < PPT; ++i) {
                    // every pair of a warp with a valid row computes (straight-line code the
                    // compiler can interleave); invalid rows produce values no valid cell reads
                    if ((wskip >> ((s - 1) * PPT + i)) & 1) {
                        val[i] = make_double2(0.0, 0.0);
                        continue;
                    }
                    const int h2 = lcell[i] >> 1;  // pair index within a plane
                    // x neighbourhood x = c-XA .. c+1+XA: XA+1 aligned pair loads, or (XSHFL)
                    // the centre pair and warp shuffles, since the lanes of a warp own
                    // consecutive pairs of a tile row. Edge lanes get values from beyond the
                    // row, exactly as the shifted loads did: those cells are never output.
                    double xs[2 * XA + 2];
                    if constexpr (XSHFL) {
                        const double2 ctr = CFG::STACK ? colw[CFG::STACK ? i + R : 0] : pc[h2];
                        const int lane = tid & 31;
#pragma unroll
                        for (int t = 0; t <= XA; ++t) {
                            const int d = t - XA / 2;
                            xs[2 * t] = d == 0 ? ctr.x : __shfl_sync(0xffffffffu, ctr.x, lane + d);
                            xs[2 * t + 1] =
                                d == 0 ? ctr.y : __shfl_sync(0xffffffffu, ctr.y, lane + d);
                            if constexpr (NARROW) {
                                // every column is an output column: the row's edge lanes take
                                // the pair beyond the warp's row from the box
                                if (d != 0 && (lane + d < 0 || lane + d > 31)) {
                                    const double2 w = pc[h2 + d];
                                    xs[2 * t] = w.x;
                                    xs[2 * t + 1] = w.y;
                                }
                            }
                        }
                    } else {
#pragma unroll
                        for (int t = 0; t <= XA; ++t) {
                            const double2 w = (CFG::STACK && t == XA / 2)
                                                  ? colw[CFG::STACK ? i + R : 0]
                                                  : pc[h2 - XA / 2 + t];
                            xs[2 * t] = w.x;
                            xs[2 * t + 1] = w.y;
                        }
                    }
                    auto X = [&](int q, int dx) -> double { return xs[q + dx + XA]; };
                    auto Yp = [&](int dy) -> double2 {
                        if constexpr (CFG::STACK) return colw[i + R + dy];
                        else return pc[h2 + dy * (LX / 2)];
                    };
                    // z neighbours of level s-1 at planes k-R .. k+R: register queue zq[s-1]
                    // holds k-R .. k+R-1 (oldest first), the newest (k+R) was produced above
                    auto Zp = [&](int dz) -> double2 {
                        if (dz == R) return newest[i];
                        if (ZPS && dz > 0)
                            return reinterpret_cast<const double2*>(
                                ring0 + vslot(R - dz) * CELLS_S)[lcell[i] >> 1];
                        return zq[s - 1][i][(dz + R + PH) % ZQD];
                    };
                    auto Cp = [&](int a) -> double2 { return aux[(a * AYX + ai[i]) >> 1]; };
                    auto comp = [](const double2& v, int q) -> double { return q ? v.y : v.x; };
                    double out[2];
                    if constexpr (KIND == K_CONST7) {
                        const double c0 = p.cc[0], c1 = p.cc[1];
                        const double2 yp = Yp(1), ym = Yp(-1), zp = Zp(1), zm = Zp(-1);
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            double v = dmul(c0, X(q, 0));
                            v = dadd(v, dmul(c1, dadd(X(q, 1), X(q, -1))));
                            v = dadd(v, dmul(c1, dadd(comp(yp, q), comp(ym, q))));
                            v = dadd(v, dmul(c1, dadd(comp(zp, q), comp(zm, q))));
                            out[q] = v;
                        }
                    } else if constexpr (KIND == K_VAR7) {
                        const double2 yp = Yp(1), ym = Yp(-1), zp = Zp(1), zm = Zp(-1);
                        double2 cf[7];
                        if (!CQ || s == 1) {
#pragma unroll
                            for (int a = 0; a < 7; ++a) cf[a] = Cp(a);
                            if constexpr (PHQ) {
#pragma unroll
                                for (int a = 0; a < 7; ++a) cqr[PHQ ? PH & 1 : 0][i][CQ ? a : 0] = cf[a];
                            } else if constexpr (CQ) {
#pragma unroll
                                for (int a = 0; a < 7; ++a) cnew[i][a] = cf[a];
                            }
                        } else if constexpr (PHQ) {  // the set level 1 filled one iteration ago
#pragma unroll
                            for (int a = 0; a < 7; ++a) cf[a] = cqr[PHQ ? (PH + 1) & 1 : 0][i][CQ ? a : 0];
                        } else {
#pragma unroll
                            for (int a = 0; a < 7; ++a) cf[a] = cq[CQ ? s - 2 : 0][i][CQ ? a : 0];
                        }
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            double v = dmul(comp(cf[0], q), X(q, 0));
                            v = dadd(v, dmul(comp(cf[1], q), X(q, 1)));
                            v = dadd(v, dmul(comp(cf[2], q), X(q, -1)));
                            v = dadd(v, dmul(comp(cf[3], q), comp(yp, q)));
                            v = dadd(v, dmul(comp(cf[4], q), comp(ym, q)));
                            v = dadd(v, dmul(comp(cf[5], q), comp(zp, q)));
                            v = dadd(v, dmul(comp(cf[6], q), comp(zm, q)));
                            out[q] = v;
                        }
                    } else if constexpr (KIND == K_CONST25) {
                        double2 yp[4], ym[4];
#pragma unroll
                        for (int r = 1; r <= 4; ++r) {
                            yp[r - 1] = Yp(r);
                            ym[r - 1] = Yp(-r);
                        }
                        const double2 cf = Cp(0);
                        // level s-2 at plane k: t0-1 from the aux ring (s = 1), else the oldest
                        // entry of level s-2's z queue (before this iteration's shift)
                        const double2 up = s == 1 ? Cp(1) : zq[s >= 2 ? s - 2 : 0][i][PH % ZQD];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const double vc = X(q, 0);
                            double lap = dmul(p.cc[0], vc);
#pragma unroll
                            for (int r = 1; r <= 4; ++r) {
                                double sr = dadd(X(q, r), X(q, -r));
                                sr = dadd(sr, comp(yp[r - 1], q));
                                sr = dadd(sr, comp(ym[r - 1], q));
                                sr = dadd(sr, comp(Zp(r), q));
                                sr = dadd(sr, comp(Zp(-r), q));
                                lap = dadd(lap, dmul(p.cc[r], sr));
                            }
                            out[q] = dadd(dsub(dmul(2.0, vc), comp(up, q)), dmul(comp(cf, q), lap));
                        }
                    } else {  // K_VAR25
                        double2 yp[4], ym[4];
#pragma unroll
                        for (int r = 1; r <= 4; ++r) {
                            yp[r - 1] = Yp(r);
                            ym[r - 1] = Yp(-r);
                        }
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            double v = dmul(comp(Cp(0), q), X(q, 0));
#pragma unroll
                            for (int r = 1; r <= 4; ++r) {
                                const int b = 3 * (r - 1);
                                v = dadd(v, dmul(comp(Cp(b + 1), q), dadd(X(q, r), X(q, -r))));
                                v = dadd(v, dmul(comp(Cp(b + 2), q),
                                                 dadd(comp(yp[r - 1], q), comp(ym[r - 1], q))));
                                v = dadd(v, dmul(comp(Cp(b + 3), q),
                                                 dadd(comp(Zp(r), q), comp(Zp(-r), q))));
                            }
                            out[q] = v;
                        }
                    }
                    val[i] = make_double2(out[0], out[1]);
                }
                // (2) ghost cells of level s hold the parity-(t0+s) field's ghosts (block edges
                //     and ghost planes only: a uniform branch elsewhere)
                if (s < TB && (plane_ghost || any_ghost_col)) {
                    const uint32_t fix = plane_ghost ? ok_mask : col_fix;
#pragma unroll
                    for (int i = 0; i < PPT; ++i) {
                        if (dyv[i] < s * R) continue;
                        if ((fix >> (2 * i)) & 1) val[i].x = gh[s < TB ? s - 1 : 0][i].x;
                        if ((fix >> (2 * i + 1)) & 1) val[i].y = gh[s < TB ? s - 1 : 0][i].y;
                    }
                }
                // (3) results: the level-s centre ring + z queue input (s < TB) or the output
                //     staging plane (s == TB)
                if (s < TB) {
                    // the centre-ring store is deferred to the end of the iteration so that
                    // the loads of every level can be scheduled ahead of it
                    ring_slot[s < TB ? s : 0] = (k + KOFF) % QL;
#pragma unroll
                    for (int i = 0; i < PPT; ++i) {
                        fresh[s < TB ? s : 0][i] = val[i];
                        newest[i] = val[i];
                    }
                } else if (k >= ug.za && k < ug.zb) {
                    if constexpr (DOUT) {
                        // straight to global memory: interior output cells only (the TMA store
                        // map's clipping, done by the masks); a full pair is one aligned
                        // 16-byte store (x pair origins are even, off + R is even)
                        double* dst = (CHAIN ? SU2[seq & 1].dst_final : p.dst_final) + (long long)k * p.plane;
                        constexpr uint32_t FULL = PPT == 16 ? 0xffffffffu : (1u << (2 * PPT)) - 1u;
                        if constexpr (!(NARROW && TB == 1) && PPT == 1) {
                            // (edge lanes of every warp hold halo or half-output pairs: no
                            // per-thread fast path, which would make every warp run both paths;
                            // measured: var7pt 1024^3 +2.7%, 384^3 +2.4%, 512^3 +1.0%; two-pair
                            // const7pt threads 512^3 -0.9%, so those keep the branch)
#pragma unroll
                            for (int i = 0; i < PPT; ++i)
                                st_pair_masked(dst + colidx[2 * i], dst + colidx[2 * i + 1], val[i],
                                               (dmask >> (2 * i)) & 3u);
                        } else if (dmask == FULL) {  // every pair whole (all threads of interior tiles)
                            if constexpr (CFG::STACK) {
                                // a thread's pairs sit in consecutive rows of one column (no
                                // clamped coordinate in a whole-pair thread): one base, row pitch
                                double* d0 = dst + colidx[0];
#pragma unroll
                                for (int i = 0; i < PPT; ++i)
                                    *reinterpret_cast<double2*>(d0 + i * p.pitch) = val[i];
                            } else {
#pragma unroll
                                for (int i = 0; i < PPT; ++i)
                                    *reinterpret_cast<double2*>(dst + colidx[2 * i]) = val[i];
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < PPT; ++i) {
                                const uint32_t m = (dmask >> (2 * i)) & 3u;
                                if (m == 3u) {
                                    *reinterpret_cast<double2*>(dst + colidx[2 * i]) = val[i];
                                } else {
                                    if (m & 1u) dst[colidx[2 * i]] = val[i].x;
                                    if (m & 2u) dst[colidx[2 * i + 1]] = val[i].y;
                                }
                            }
                        }
                    } else {
                    double* stg = stage + (g % 3) * STAGE;
#pragma unroll
                    for (int i = 0; i < PPT; ++i) {
                        if ((out_mask >> (2 * i)) & 1) stg[sidx[i]] = val[i].x;  // clipped by omap
                        if ((out_mask >> (2 * i + 1)) & 1) stg[sidx[i] + 1] = val[i].y;
                    }
                    }
                    if (!DOUT && any_odd_col && k >= p.zout_lo && k < p.zout_hi) {
                        double* dst = (CHAIN ? SU2[seq & 1].dst_final : p.dst_final) + (long long)k * p.plane;
#pragma unroll
                        for (int i = 0; i < PPT; ++i) {
                            if ((odd_mask >> (2 * i)) & 1) dst[colidx[2 * i]] = val[i].x;
                            if ((odd_mask >> (2 * i + 1)) & 1) dst[colidx[2 * i + 1]] = val[i].y;
                        }
                    }
                    if (CHAIN ? (uflags & 1) != 0 : has_penult_1) {  // final pass only:
                        // level TB-1 of the same cells
                        double* pen = (CHAIN ? SU2[seq & 1].dst_penult : p.dst_penult) + (long long)k * p.plane;
#pragma unroll
                        for (int i = 0; i < PPT; ++i) {
                            // level TB-1 at plane k
                            const double2 c2 = ZPS ? ctrk[ZPS ? i : 0] : zq[TB - 1][i][ZPS ? 0 : (R + PH) % ZQD];
                            const int b = 2 * i;
                            if ((out_mask >> b) & 1 && !((ghost_mask >> b) & 1)) pen[colidx[b]] = c2.x;
                            if ((out_mask >> (b + 1)) & 1 && !((ghost_mask >> (b + 1)) & 1))
                                pen[colidx[b + 1]] = c2.y;
                        }
                    }
                    if (INSTR && p.ledger) {  // instrumentation: this unit owns these updates
                        const int kz = k + p.zoff - R;
                        if (kz >= 0 && kz < p.nzg) {
#pragma unroll
                            for (int i = 0; i < PPT; ++i)
#pragma unroll
                                for (int q = 0; q < 2; ++q) {
                                    const int b = 2 * i + q;
                                    if (!((out_mask >> b) & 1) || ((ghost_mask >> b) & 1)) continue;
                                    const int xa = xa0 + cell_lx(i) + q, ya = ya0 + cell_ly(i);
                                    const long long cell = ((long long)kz * p.ny + (ya - R)) * p.nx + (xa - R);
                                    for (int s2 = 0; s2 < TB; ++s2)
                                        atomicAdd(p.ledger + (long long)(p.ledger_t + s2) * p.nzg * p.ny * p.nx + cell, 1u);
                                }
                        }
                    }
                    if (!CHAIN && p.push_hz > 0) {  // (push_hz = 0: no neighbour slabs)
                        // halo push: boundary planes go to the neighbour slab as they are made
                        const bool dn = p.push_dn_final && k < p.zout_lo + p.push_hz;
                        const bool up = p.push_up_final && k >= p.zout_hi - p.push_hz;
                        // (a thin slab's plane may belong to both neighbours' halos)
#pragma unroll
                        for (int side = 0; side < 2; ++side) {
                            if (!(side ? up : dn)) continue;
                            const long long o =
                                (long long)k * p.plane + (side ? p.push_up_off : p.push_dn_off);
                            double* fin = (side ? p.push_up_final : p.push_dn_final) + o;
                            double* pen = has_penult_1
                                              ? (side ? p.push_up_penult : p.push_dn_penult) + o
                                              : nullptr;
                            // a full pair is one aligned 16-byte store (the neighbour's buffers
                            // share this layout and the offsets are whole planes), so a warp's
                            // push is 512 contiguous bytes of NVLink writes, not 32 strided
                            // 8-byte ones per cell of the pair. Radius 4: scalar stores (the
                            // vector path cost the 255-register const25pt kernel a spill)
                            constexpr bool PUSH_VEC = R == 1;
#pragma unroll
                            for (int i = 0; i < PPT; ++i) {
                                const double2 c2 =
                                    ZPS ? ctrk[ZPS ? i : 0] : zq[TB - 1][i][ZPS ? 0 : (R + PH) % ZQD];
                                const uint32_t m = ((out_mask & ~ghost_mask) >> (2 * i)) & 3u;
                                if (PUSH_VEC && m == 3u) {
                                    *reinterpret_cast<double2*>(fin + colidx[2 * i]) = val[i];
                                    if (pen) *reinterpret_cast<double2*>(pen + colidx[2 * i]) = c2;
                                } else {
#pragma unroll
                                    for (int q = 0; q < 2; ++q) {
                                        if (!((m >> q) & 1u)) continue;
                                        fin[colidx[2 * i + q]] = q ? val[i].y : val[i].x;
                                        if (pen) pen[colidx[2 * i + q]] = q ? c2.y : c2.x;
                                    }
                                }
                            }
                        }
                    }
                    staged = !DOUT;
                }
            }
            if constexpr (CSYNC)
                if (!cwaited) cluster_wait();
            // deferred centre-ring stores of levels 1..TB-1 (read by other threads from the
            // next iteration on, behind the barrier)
#pragma unroll
            for (int L = 1; L < TB; ++L) {
                if (ring_slot[L] < 0) continue;
                double2* wr = reinterpret_cast<double2*>(ringL + ((L - 1) * QL + ring_slot[L]) * CELLS_S);
#pragma unroll
                for (int i = 0; i < PPT; ++i) wr[lcell[i] >> 1] = fresh[L][i];
                if constexpr (CY > 1) {
                    // the R own rows next to an inner edge also go into the neighbour's ring,
                    // as the rows beyond its edge (same slot and column, row shifted by OWN)
#pragma unroll
                    for (int i = 0; i < PPT; ++i) {
                        const int ly = lcell[i] / LX;
                        if (!lo_edge && ly < 2 * R)
                            st_cluster_d2(mapa_rank(smem_u32(&wr[(lcell[i] + OWN * LX) >> 1]), crank - 1),
                                          fresh[L][i]);
                        if (!hi_edge && ly >= LY - 2 * R)
                            st_cluster_d2(mapa_rank(smem_u32(&wr[(lcell[i] - OWN * LX) >> 1]), crank + 1),
                                          fresh[L][i]);
                    }
                }
            }
            if constexpr (CSYNC)
                cluster_arrive();  // this iteration's ring rows are complete
            // advance every level's z queue by one plane (and the coefficient queue)
            if constexpr (CQ && !PHQ) {
#pragma unroll
                for (int L = CQD - 1; L > 0; --L)
#pragma unroll
                    for (int i = 0; i < PPT; ++i)
#pragma unroll
                        for (int a = 0; a < CQN; ++a) cq[L][i][a] = cq[L - 1][i][a];
#pragma unroll
                for (int i = 0; i < PPT; ++i)
#pragma unroll
                    for (int a = 0; a < CQN; ++a) cq[0][i][a] = cnew[i][a];
            }
#pragma unroll
            for (int L = 0; L < TB; ++L) {
#pragma unroll
                for (int i = 0; i < PPT; ++i) {
                    if constexpr (PHZ) {
                        zq[L][i][PH % ZQD] = fresh[L][i];  // the oldest entry's slot
                    } else {
#pragma unroll
                        for (int d = 0; d + 1 < ZQD; ++d) zq[L][i][d] = zq[L][i][d + 1];
                        zq[L][i][ZQD - 1] = fresh[L][i];
                    }
                }
            }
            if (tr) trp[2] = clock64();
            // hand the staged output plane to the async proxy; the store thread issues it next
            // iteration
            if (staged) {
                fence_proxy_async_smem();
                if (tid == STORE_TID) {
                    pend = true;
                    pend_x = ug.tx * p.ox;
                    pend_y = ug.ty * OYC + crank * OWN + oy_lo - H;
                    pend_z = j - H - p.oz0;
                    pend_b = int(g % 3);
                    if constexpr (CHAIN) pend_q = uflags >> 1;
                }
            }
            if constexpr (CHAIN)
                if (tid == STORE_TID && it == n_it - 1) pub_next = u;  // unit finished
            // instrumentation: one record per unit (a cluster's unit by its leader CTA)
            if (INSTR && p.trace && tid == 0 && crank == 0) {
                if (it == 0) unit_t0 = global_ns();
                if (it == n_it - 1) {
                    const unsigned long long r = atomicAdd(p.trace_n, 1ull);
                    if ((long long)r < p.trace_cap) {
                        unsigned long long* rec = p.trace + 4 * r;
                        rec[0] = ((unsigned long long)p.trace_pass << 32) | unsigned(u + p.unit0);
                        rec[1] = ((unsigned long long)blockIdx.x << 32) | sm_id();
                        rec[2] = unit_t0;
                        rec[3] = global_ns();
                    }
                }
            }
            // three staging planes: the plane the next iteration writes was handed to the store
            // issued two iterations ago, so only that older store must have finished reading
            if (tid == STORE_TID) {
                if (stored_now)
                    bulk_wait_read_but1();  // the store issued this iteration may stay in flight
                else
                    bulk_wait_read_all();
            }
            if (tr) trp[3] = clock64();
            ++g;
            if (++gs == NR0) {
                gs = 0;
                gph ^= 1u;
            }
            if constexpr (NAR > 0) {
                if (++as == NAR) {
                    as = 0;
                    aph ^= 1u;
                }
            }
        };
        constexpr int NPH = PHZ ? ZQD : 1;
        for (int it0 = 0; it0 < n_it; it0 += NPH) {
            auto phase = [&](auto PHc) -> bool {
                if (it0 + decltype(PHc)::value >= n_it) return false;
                iteration(PHc, it0 + decltype(PHc)::value);
                return true;
            };
            unroll_phases<0, NPH>(phase);
        }
        if constexpr (!CHAIN && CY == 1 && GIRIH_IPC_FLAGS) {
            // IPC z-slabs: the last boundary unit of the pass signals the neighbours
            if (p.bflag_n > 0 && u < p.bflag_n) {
                __syncthreads();  // every thread's peer stores of this unit are issued
                if (tid == 0) {
                    __threadfence_system();  // cumulative: the CTA's pushes before the count
                    const int old = atomicAdd(p.bdone, 1);
                    if (old == p.bdone_base + p.bflag_n - 1) {
                        __threadfence_system();  // every pushing CTA's stores before the flags
                        if (p.bflag_dn)
                            asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p.bflag_dn),
                                         "r"(p.bflag_val) : "memory");
                        if (p.bflag_up)
                            asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p.bflag_up),
                                         "r"(p.bflag_val) : "memory");
                    }
                }
            }
        }
    }
    if constexpr (PACE) {
        // the last iteration's arrival (a neighbour may still wait for it), then no CTA leaves
        // while a neighbour may still arrive on its barriers
        if (tid == 0 && g > G0) pace_arrive(g - G0 - 1);
        cluster_arrive();
        cluster_wait();
    } else if constexpr (CY > 1) {
        cluster_wait();  // no CTA leaves while a neighbour may push into it
    }
    __syncthreads();
    if (tid == STORE_TID) {
        if (pend) {
            const PassDesc& od = cd.d[CHAIN ? cd.pidx[pend_q] : 0];
            tma_store_plane((CY > 1 && !lo_edge && !hi_edge) ? &od.omap_in : &od.omap,
                            stage + pend_b * STAGE, pend_x, pend_y, pend_z);
            bulk_commit();
        }
        bulk_wait_all();
        if constexpr (CHAIN)  // other CTAs may be waiting for this CTA's last unit
            if (pub_next >= 0) chain_publish(p, cd.done, pub_next);
    }
}

}  // namespace girih_gpu
