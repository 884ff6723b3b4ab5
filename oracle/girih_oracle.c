/* girih_oracle.c -- TEST INFRASTRUCTURE ONLY (see girih_oracle.h).
 *
 * Plain-C restatement of the reference CPU algorithm, compiled with
 * -ffp-contract=off exactly like the reference core (proj/CMakeLists.txt:24-25) so
 * every multiply and add rounds separately in the reference's association order.
 */
#include "girih_oracle.h"

#include <stddef.h>
#include <string.h>

typedef struct {
    int radius, nd, flops, torder, ncoeff;
} orc_traits_t;

/* proj/src/stencil.cpp:11-17 */
static const orc_traits_t kTraits[4] = {
    {1, 2, 7, 1, 0},
    {1, 9, 13, 1, 7},
    {4, 3, 33, 2, 1},
    {4, 15, 37, 1, 13},
};

int orc_traits(int kind, int* radius, int* nd, int* flops, int* torder, int* ncoeff) {
    if (kind < 0 || kind > 3) return -1;
    const orc_traits_t* t = &kTraits[kind];
    if (radius) *radius = t->radius;
    if (nd) *nd = t->nd;
    if (flops) *flops = t->flops;
    if (torder) *torder = t->torder;
    if (ncoeff) *ncoeff = t->ncoeff;
    return 0;
}

/* proj/src/stencil.cpp:19-24 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* proj/src/stencil.cpp:49-56: five chained mixes keyed on (seed, field, k, j, i);
 * the coordinates enter as zero-extended 32-bit values. */
double orc_init_value(uint64_t seed, int field, int k, int j, int i) {
    uint64_t h = orc_splitmix64(seed ^ 0x6A09E667F3BCC909ull);
    h = orc_splitmix64(h ^ (uint64_t)field);
    h = orc_splitmix64(h ^ (uint64_t)(uint32_t)k);
    h = orc_splitmix64(h ^ (uint64_t)(uint32_t)j);
    h = orc_splitmix64(h ^ (uint64_t)(uint32_t)i);
    return (double)(h >> 11) * 0x1.0p-53 - 0.5;
}

void orc_fill_field(double* f, int X, int Y, int Z, uint64_t seed, int field) {
#pragma omp parallel for schedule(static)
    for (int k = 0; k < Z; ++k)
        for (int j = 0; j < Y; ++j) {
            double* row = f + ((size_t)k * Y + j) * X;
            for (int i = 0; i < X; ++i) row[i] = orc_init_value(seed, field, k, j, i);
        }
}

/* proj/src/stencil.cpp:58-85 (field ids: u=0, v=1, coeff c=2+c, scalars 64) */
int orc_init_state(int kind, int nx, int ny, int nz, int pad_x, uint64_t seed, double* u,
                   double* v, double* const* coeffs, double* cc) {
    int R, nc;
    if (orc_traits(kind, &R, NULL, NULL, NULL, &nc) != 0) return -1;
    const int m = 2 * R + 1;
    if (nx < m || ny < m || nz < m || pad_x < 0) return -1;
    const int X = nx + 2 * R + pad_x, Y = ny + 2 * R, Z = nz + 2 * R;
    orc_fill_field(u, X, Y, Z, seed, 0);
    orc_fill_field(v, X, Y, Z, seed, 1);
    for (int c = 0; c < nc; ++c) orc_fill_field(coeffs[c], X, Y, Z, seed, 2 + c);
    for (int c = 0; c < 5; ++c) cc[c] = orc_init_value(seed, 64, 0, 0, c);
    return 0;
}

static void remap_array(double* f, size_t n, double scale) {
#pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; ++q) f[q] = (f[q] + 0.5) * scale;
}

/* SURVEY.md 8(d) "Input remap": exact affine maps of the reference [-0.5,0.5) init onto
 * the BASELINE.json value distributions. */
void orc_apply_remap(int kind, int nx, int ny, int nz, int pad_x, double* u, double* v,
                     double* const* coeffs, double* cc) {
    int R, nc;
    if (orc_traits(kind, &R, NULL, NULL, NULL, &nc) != 0) return;
    const size_t n = (size_t)(nx + 2 * R + pad_x) * (size_t)(ny + 2 * R) * (size_t)(nz + 2 * R);
#pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; ++q) {
        u[q] = u[q] + 0.5;
        v[q] = v[q] + 0.5;
    }
    switch (kind) {
    case ORC_CONST7PT:
        cc[0] = (cc[0] + 0.5) * 0.2;
        cc[1] = (cc[1] + 0.5) * 0.2;
        break;
    case ORC_VAR7PT:
        for (int c = 0; c < nc; ++c) remap_array(coeffs[c], n, 0.14);
        break;
    case ORC_CONST25PT: {
        remap_array(coeffs[0], n, 1.0);
        double r[5];
        for (int c = 0; c < 5; ++c) r[c] = cc[c] + 0.5;
        const double s = 0.99 / (r[0] + 6 * (r[1] + r[2] + r[3] + r[4]));
        for (int c = 0; c < 5; ++c) cc[c] = r[c] * s;
        break;
    }
    case ORC_VAR25PT:
        for (int c = 0; c < nc; ++c) remap_array(coeffs[c], n, 1.0 / 26);
        break;
    }
}

/* ---- point kernels: proj/include/girih/kernels.hpp:31-85, same association ---- */

static inline double pt_const7(const double* V, size_t c, size_t sy, size_t sz, double c0,
                               double c1) {
    return c0 * V[c] + c1 * (V[c + 1] + V[c - 1]) + c1 * (V[c + sy] + V[c - sy]) +
           c1 * (V[c + sz] + V[c - sz]);
}

static inline double pt_var7(const double* V, size_t c, size_t sy, size_t sz,
                             const double* const* C) {
    return C[0][c] * V[c] + C[1][c] * V[c + 1] + C[2][c] * V[c - 1] + C[3][c] * V[c + sy] +
           C[4][c] * V[c - sy] + C[5][c] * V[c + sz] + C[6][c] * V[c - sz];
}

static inline double pt_const25(const double* V, const double* U, const double* C, size_t c,
                                size_t sy, size_t sz, const double* cc) {
    double lap = cc[0] * V[c];
    for (int r = 1; r <= 4; ++r) {
        /* one bracket per radius, six terms summed left to right (kernels.hpp:56-67) */
        const double s = V[c + r] + V[c - r] + V[c + r * sy] + V[c - r * sy] + V[c + r * sz] +
                         V[c - r * sz];
        lap = lap + cc[r] * s;
    }
    return 2 * V[c] - U[c] + C[c] * lap;
}

static inline double pt_var25(const double* V, size_t c, size_t sy, size_t sz,
                              const double* const* C) {
    double acc = C[0][c] * V[c];
    for (int r = 1; r <= 4; ++r) {
        const int b = 3 * (r - 1);
        acc = acc + C[b + 1][c] * (V[c + r] + V[c - r]);
        acc = acc + C[b + 2][c] * (V[c + r * sy] + V[c - r * sy]);
        acc = acc + C[b + 3][c] * (V[c + r * sz] + V[c - r * sz]);
    }
    return acc;
}

static double eval_point(int kind, const double* V, const double* U, const double* const* C,
                         const double* cc, size_t c, size_t sy, size_t sz) {
    switch (kind) {
    case ORC_CONST7PT: return pt_const7(V, c, sy, sz, cc[0], cc[1]);
    case ORC_VAR7PT: return pt_var7(V, c, sy, sz, C);
    case ORC_CONST25PT: return pt_const25(V, U, C[0], c, sy, sz, cc);
    default: return pt_var25(V, c, sy, sz, C);
    }
}

/* proj/src/stencil.cpp:115-127 with update_row (kernels.hpp:89-119): level t lives in u
 * when t is even, v when odd; step t reads src(t) and writes dst(t). */
long orc_naive_sweep(int kind, int nx, int ny, int nz, int pad_x, double* u, double* v,
                     const double* const* coeffs, const double* cc, long t_current, long steps) {
    int R;
    if (steps < 0 || orc_traits(kind, &R, NULL, NULL, NULL, NULL) != 0) return -1;
    const size_t X = (size_t)(nx + 2 * R + pad_x), Y = (size_t)(ny + 2 * R);
    const size_t sy = X, sz = X * Y;
    for (long t = t_current; t < t_current + steps; ++t) {
        const double* V = (t % 2 == 0) ? u : v;
        double* U = (t % 2 == 0) ? v : u;
        for (int k = R; k < R + nz; ++k)
            for (int j = R; j < R + ny; ++j) {
                const size_t row = (size_t)k * sz + (size_t)j * sy;
                for (int i = R; i < R + nx; ++i) {
                    const size_t c = row + (size_t)i;
                    U[c] = eval_point(kind, V, U, coeffs, cc, c, sy, sz);
                }
            }
    }
    return t_current + steps;
}

double orc_apply_point(int kind, int nx, int ny, int nz, int pad_x, const double* u,
                       const double* v, const double* const* coeffs, const double* cc,
                       long t_current, int i, int j, int k) {
    int R;
    (void)nz;
    if (orc_traits(kind, &R, NULL, NULL, NULL, NULL) != 0) return 0.0;
    const size_t X = (size_t)(nx + 2 * R + pad_x), Y = (size_t)(ny + 2 * R);
    const double* V = (t_current % 2 == 0) ? u : v;
    const double* U = (t_current % 2 == 0) ? v : u;
    const size_t c = ((size_t)k * Y + (size_t)j) * X + (size_t)i;
    return eval_point(kind, V, U, coeffs, cc, c, X, X * Y);
}

/* proj/src/stencil.cpp:129-146: FNV-1a over the little-endian bytes of interior doubles */
uint64_t orc_interior_checksum(const double* f, int nx, int ny, int nz, int pad_x, int R) {
    const size_t X = (size_t)(nx + 2 * R + pad_x), Y = (size_t)(ny + 2 * R);
    uint64_t h = 0xCBF29CE484222325ull;
    for (int k = R; k < R + nz; ++k)
        for (int j = R; j < R + ny; ++j)
            for (int i = R; i < R + nx; ++i) {
                uint64_t bits;
                memcpy(&bits, &f[((size_t)k * Y + j) * X + i], sizeof bits);
                for (int b = 0; b < 8; ++b) {
                    h ^= (bits >> (8 * b)) & 0xFF;
                    h *= 0x100000001B3ull;
                }
            }
    return h;
}

uint64_t orc_fnv_all(const double* f, uint64_t n) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (uint64_t q = 0; q < n; ++q) {
        uint64_t bits;
        memcpy(&bits, &f[q], sizeof bits);
        for (int b = 0; b < 8; ++b) {
            h ^= (bits >> (8 * b)) & 0xFF;
            h *= 0x100000001B3ull;
        }
    }
    return h;
}

/* Row digest: FNV-1a of every row's bytes (rows of row_elems doubles, in k, j order), then
 * FNV-1a over the little-endian bytes of those row hashes. Test helper: a checksum of
 * checksums that a GPU can also compute in parallel, one thread per row (girih_gpu_row_digest). */
uint64_t orc_row_digest(const double* f, uint64_t nrows, uint64_t row_elems) {
    uint64_t d = 0xCBF29CE484222325ull;
    for (uint64_t r = 0; r < nrows; ++r) {
        const uint64_t h = orc_fnv_all(f + r * row_elems, row_elems);
        for (int b = 0; b < 8; ++b) {
            d ^= (h >> (8 * b)) & 0xFF;
            d *= 0x100000001B3ull;
        }
    }
    return d;
}
