// zwave.cuh -- the temporally-blocked z-wavefront stencil pass for sm_100a.
//
// One launch advances a z-slab (or the whole grid) by TB time steps in a single HBM pass.
// It is the B200 counterpart of the reference's multi-core wavefront diamond engine
// (proj/src/engine.cpp:203-260): there a thread group shares one cache block and sweeps z
// with a pipelined wavefront; here a CTA owns an (x,y) tile column and streams its z-planes
// through shared memory:
//
//   * level 0 (the input time level) arrives plane by plane by TMA (cp.async.bulk.tensor,
//     box LX x LY x 1) into a ring of NR0 = 2R+1+P planes completed on mbarriers, P planes
//     ahead of use -- the z-wavefront;
//   * level s (1..TB) of plane k_s = j - s*R is computed at global iteration j from level
//     s-1 planes k_s-R .. k_s+R: x/y/z neighbours come from the level-(s-1) smem ring, the
//     newest plane (k_s+R) from the register the same thread produced one level earlier;
//   * levels 1..TB-1 are kept in per-level rings of 2R+1 planes; level TB is stored to HBM;
//   * the tile shrinks by R per side per level (overlapped / trapezoid tiling in x and y,
//     and in z at z-chunk boundaries), so no inter-CTA synchronisation exists inside a pass;
//     the x halo is H or H+1 so that every TMA box starts on a 16-byte boundary.
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
    int units;               // tiles_x * tiles_y * nzc
    int hx, ox;              // x halo (H or H+1) and output tile width LX - 2*hx: TMA needs the
                             // innermost box coordinate 16-byte aligned (even for fp64)
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
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

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Work-unit cursor: unit u -> (tile x, tile y, z chunk); a unit's level-0 stream covers
// planes [za - H, zb + H).
struct UnitGeom {
    int tx, ty, za, zb;
};

__device__ __forceinline__ UnitGeom unit_geom(const PassParams& p, int u) {
    UnitGeom g;
    g.tx = u % p.tiles_x;
    const int r = u / p.tiles_x;
    g.ty = r % p.tiles_y;
    const int zc = r / p.tiles_y;
    g.za = p.zout_lo + zc * p.zc_len;
    g.zb = min(g.za + p.zc_len, p.zout_hi);
    return g;
}

template <int KIND, int TB, int LX, int LY, int NT, int P>
struct ZwaveConfig {
    static constexpr int R = KindTraits<KIND>::R;
    static constexpr int Q = 2 * R + 1;     // z window of one level
    static constexpr int NR0 = Q + P;       // level-0 TMA ring depth
    static constexpr int H = TB * R;        // halo of the loaded tile
    static constexpr int OX = LX - 2 * H;   // output tile
    static constexpr int OY = LY - 2 * H;
    static constexpr int CELLS = LX * LY;
    static constexpr int CPT = CELLS / NT;  // cells per thread
    static constexpr int NRING = NR0 + (TB - 1) * Q;
    static constexpr size_t SMEM = size_t(NRING) * CELLS * sizeof(double) + NR0 * sizeof(uint64_t);
    static_assert(CELLS % NT == 0, "tile must split evenly over the CTA");
    static_assert(OX - 2 > 0 && OY > 0, "tile too small for the halo (x halo may be H+1)");
    static_assert(LX <= 256 && LY <= 256, "TMA box limit");
    static_assert((LX * 8) % 16 == 0, "TMA inner box must be a multiple of 16 bytes");
};

template <int KIND, int TB, int LX, int LY, int NT, int P>
__global__ void __launch_bounds__(NT, 1)
    zwave_kernel(const __grid_constant__ CUtensorMap src_map,
                 const __grid_constant__ PassParams p) {
    using CFG = ZwaveConfig<KIND, TB, LX, LY, NT, P>;
    constexpr int R = CFG::R, Q = CFG::Q, NR0 = CFG::NR0, H = CFG::H;
    constexpr int CELLS = CFG::CELLS, CPT = CFG::CPT;
    constexpr int OY = CFG::OY;
    constexpr uint32_t PLANE_BYTES = CELLS * sizeof(double);
    // large multiples keep ring indices non-negative for planes below 0
    constexpr int KOFF = Q * 4096;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring0 = reinterpret_cast<double*>(smem_raw);
    double* ringL = ring0 + NR0 * CELLS;  // level s (1..TB-1) ring at ringL + (s-1)*Q*CELLS
    uint64_t* mbar = reinterpret_cast<uint64_t*>(ringL + (TB - 1) * Q * CELLS);

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < NR0; ++b) mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    // ---- producer cursor (thread 0): element index g -> (unit, iteration) ----
    // Global stream counter starts at a multiple of NR0 so that early (g - 2R) indices stay
    // non-negative and the first phase parity is 0.
    constexpr long long G0 = 4LL * NR0;
    int pu = blockIdx.x;          // producer's unit
    int pit = 0;                  // producer's iteration within the unit
    UnitGeom pg{};
    if (pu < p.units) pg = unit_geom(p, pu);
    long long pgidx = G0;         // global index of the next element to load

    auto producer_issue = [&](void) {
        // issue the load for element pgidx, then advance the cursor
        if (pu >= p.units) return;
        const int j = pg.za - H + pit;
        const int slot = int(pgidx % NR0);
        const int xd = p.off + pg.tx * p.ox + R - p.hx;  // even by construction
        const int yd = pg.ty * OY + R - H;
        mbar_arrive_expect_tx(&mbar[slot], PLANE_BYTES);
        tma_load_plane(ring0 + slot * CELLS, &src_map, xd, yd, j, &mbar[slot]);
        ++pgidx;
        ++pit;
        if (pit >= (pg.zb - pg.za) + 2 * H) {
            pit = 0;
            pu += gridDim.x;
            if (pu < p.units) pg = unit_geom(p, pu);
        }
    };

    if (tid == 0)
        for (int e = 0; e < P; ++e) producer_issue();

    // ---- per-thread cell constants ----
    int lcell[CPT], dmin[CPT];
    bool out_col[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
        const int c = tid + NT * i;
        lcell[i] = c;
        const int lx = c % LX, ly = c / LX;
        const int dx = min(lx, LX - 1 - lx), dy = min(ly, LY - 1 - ly);
        dmin[i] = min(dx, dy);
        out_col[i] = dx >= p.hx && dy >= H;
    }

    long long g = G0;  // consumer's global element index
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const UnitGeom ug = unit_geom(p, u);
        const int n_it = (ug.zb - ug.za) + 2 * H;
        const int xa0 = ug.tx * p.ox + R - p.hx;  // allocated x of local lx = 0
        const int ya0 = ug.ty * OY + R - H;

        // per-cell column data for this unit
        int xa[CPT], ya[CPT];
        bool col_alloc[CPT], col_ghost[CPT];
        long long colidx[CPT];
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const int lx = lcell[i] % LX, ly = lcell[i] / LX;
            xa[i] = xa0 + lx;
            ya[i] = ya0 + ly;
            col_alloc[i] = xa[i] >= 0 && xa[i] < p.X && ya[i] >= 0 && ya[i] < p.Y;
            col_ghost[i] = xa[i] < R || xa[i] >= R + p.nx || ya[i] < R || ya[i] >= R + p.ny;
            const int cx = min(max(xa[i], 0), p.X - 1), cy = min(max(ya[i], 0), p.Y - 1);
            colidx[i] = (long long)cy * p.pitch + p.off + cx;
        }

        for (int it = 0; it < n_it; ++it, ++g) {
            const int j = ug.za - H + it;  // level-0 plane of this iteration
            __syncthreads();               // previous iteration's smem traffic is complete
            if (tid == 0) producer_issue();
            {
                const int slot = int(g % NR0);
                mbar_wait(&mbar[slot], uint32_t((g / NR0) & 1));
            }

            // uniform per-level plane data
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
                double newest = 0.0;  // level s-1 value at (cell, k_s + R)
#pragma unroll
                for (int s = 1; s <= TB; ++s) {
                    const int k = j - s * R;  // plane of level s
                    // lower bounds are monotone in s (higher levels sit on lower planes)
                    if (it < 2 * s * R || k < 0) break;  // uniform
                    if (dmin[i] < s * R) break;  // column outside level-s valid area
                    if (!col_alloc[i]) break;
                    // above the buffer: skip this level only; level s+1 sits R planes lower
                    // (a ghost plane there, so it never reads this level's value)
                    if (k >= p.Zloc) continue;
                    const int kg = k + p.zoff;
                    const bool plane_ghost = kg < R || kg >= R + p.nzg;
                    const long long gidx = (long long)k * p.plane + colidx[i];

                    // pointers to the level-(s-1) planes k-R .. k+R (dz index 0..2R)
                    const double* pl[Q];
                    if (s == 1) {
#pragma unroll
                        for (int d = 0; d < Q; ++d)
                            pl[d] = ring0 + int((g - 2 * R + d) % NR0) * CELLS;
                    } else {
                        const double* base = ringL + (s - 2) * Q * CELLS;
#pragma unroll
                        for (int d = 0; d < Q; ++d)
                            pl[d] = base + ((k - R + d + KOFF) % Q) * CELLS;
                    }
                    const int c = lcell[i];
                    auto V = [&](int dx, int dy, int dz) -> double {
                        if (dz == R && s > 1) return newest;
                        return pl[dz + R][c + dx + dy * LX];
                    };

                    double val;
                    if (plane_ghost || col_ghost[i]) {
                        val = __ldg(&p.ghost[(p.parity0 + s) & 1][gidx]);
                    } else if constexpr (KIND == K_CONST7) {
                        const double c0 = p.cc[0], c1 = p.cc[1];
                        val = dmul(c0, V(0, 0, 0));
                        val = dadd(val, dmul(c1, dadd(V(1, 0, 0), V(-1, 0, 0))));
                        val = dadd(val, dmul(c1, dadd(V(0, 1, 0), V(0, -1, 0))));
                        val = dadd(val, dmul(c1, dadd(V(0, 0, 1), V(0, 0, -1))));
                    } else if constexpr (KIND == K_VAR7) {
                        val = dmul(__ldg(&p.coeff[0][gidx]), V(0, 0, 0));
                        val = dadd(val, dmul(__ldg(&p.coeff[1][gidx]), V(1, 0, 0)));
                        val = dadd(val, dmul(__ldg(&p.coeff[2][gidx]), V(-1, 0, 0)));
                        val = dadd(val, dmul(__ldg(&p.coeff[3][gidx]), V(0, 1, 0)));
                        val = dadd(val, dmul(__ldg(&p.coeff[4][gidx]), V(0, -1, 0)));
                        val = dadd(val, dmul(__ldg(&p.coeff[5][gidx]), V(0, 0, 1)));
                        val = dadd(val, dmul(__ldg(&p.coeff[6][gidx]), V(0, 0, -1)));
                    } else if constexpr (KIND == K_CONST25) {
                        const double vc = V(0, 0, 0);
                        double lap = dmul(p.cc[0], vc);
#pragma unroll
                        for (int r = 1; r <= 4; ++r) {
                            double sr = dadd(V(r, 0, 0), V(-r, 0, 0));
                            sr = dadd(sr, V(0, r, 0));
                            sr = dadd(sr, V(0, -r, 0));
                            sr = dadd(sr, V(0, 0, r));
                            sr = dadd(sr, V(0, 0, -r));
                            lap = dadd(lap, dmul(p.cc[r], sr));
                        }
                        // level s-2 at the centre: t0-1 from src_prev, else the level-(s-2) ring
                        double uprev;
                        if (s == 1) {
                            uprev = p.src_prev[gidx];
                        } else if (s == 2) {
                            uprev = ring0[int((g - 2 * R) % NR0) * CELLS + c];
                        } else {
                            const double* b2 = ringL + (s - 3) * Q * CELLS;
                            uprev = b2[((k + KOFF) % Q) * CELLS + c];
                        }
                        val = dadd(dsub(dmul(2.0, vc), uprev),
                                   dmul(__ldg(&p.coeff[0][gidx]), lap));
                    } else {  // K_VAR25
                        val = dmul(__ldg(&p.coeff[0][gidx]), V(0, 0, 0));
#pragma unroll
                        for (int r = 1; r <= 4; ++r) {
                            const int b = 3 * (r - 1);
                            val = dadd(val, dmul(__ldg(&p.coeff[b + 1][gidx]),
                                                 dadd(V(r, 0, 0), V(-r, 0, 0))));
                            val = dadd(val, dmul(__ldg(&p.coeff[b + 2][gidx]),
                                                 dadd(V(0, r, 0), V(0, -r, 0))));
                            val = dadd(val, dmul(__ldg(&p.coeff[b + 3][gidx]),
                                                 dadd(V(0, 0, r), V(0, 0, -r))));
                        }
                    }

                    if (s < TB) {
                        ringL[((s - 1) * Q + (k + KOFF) % Q) * CELLS + c] = val;
                        newest = val;
                    } else {
                        // level TB: output tile cells of interior planes [za, zb)
                        if (out_col[i] && !col_ghost[i] && k >= ug.za && k < ug.zb) {
                            p.dst_final[gidx] = val;
                            if (p.dst_penult) p.dst_penult[gidx] = V(0, 0, 0);
                        }
                    }
                }
            }
        }
    }
}

}  // namespace girih_gpu
