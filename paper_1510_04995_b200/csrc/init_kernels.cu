// init_kernels.cu -- device-side counter-based initialisation and FP64 rate probe.
//
// init_value (proj/src/stencil.cpp:19-24, 49-56) is pure 64-bit integer mixing plus an exact
// conversion, so the device reproduces the host generator bit for bit; each GPU fills its own
// z-slab (keyed on global (k, j, i)) without any host fill or H2D of the state.
#include <cstdint>

#include "device_api.h"

namespace girih_gpu {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ double init_value_dev(uint64_t seed, int field, int k, int j, int i) {
    uint64_t h = splitmix64(seed ^ 0x6A09E667F3BCC909ull);
    h = splitmix64(h ^ static_cast<uint64_t>(field));
    h = splitmix64(h ^ static_cast<uint64_t>(static_cast<uint32_t>(k)));
    h = splitmix64(h ^ static_cast<uint64_t>(static_cast<uint32_t>(j)));
    h = splitmix64(h ^ static_cast<uint64_t>(static_cast<uint32_t>(i)));
    return __dsub_rn(__dmul_rn(static_cast<double>(h >> 11), 0x1.0p-53), 0.5);
}

// Fills local planes [0, Zloc) of a device-layout buffer. Global allocated plane of local
// plane k is k + zoff; cells outside the global allocation are left untouched.
__global__ void init_field_kernel(double* buf, int pitch, int off, int X, int Y, int Zloc,
                                  int zoff, int Zg, uint64_t seed, int field, int remap,
                                  double scale) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    if (i >= X || j >= Y || k >= Zloc) return;
    const int kg = k + zoff;
    if (kg < 0 || kg >= Zg) return;
    double v = init_value_dev(seed, field, kg, j, i);
    // SURVEY.md 8(d) remap: fields x + 0.5 (scale 1), coefficient grids (x + 0.5) * scale
    if (remap) v = __dmul_rn(__dadd_rn(v, 0.5), scale);
    buf[(static_cast<long long>(k) * Y + j) * pitch + off + i] = v;
}

cudaError_t launch_init_field(double* buf, int pitch, int off, int X, int Y, int Zloc, int zoff,
                              int Zg, uint64_t seed, int field, int remap, double scale,
                              cudaStream_t stream) {
    dim3 block(128);
    dim3 grid((X + 127) / 128, Y, Zloc);
    init_field_kernel<<<grid, block, 0, stream>>>(buf, pitch, off, X, Y, Zloc, zoff, Zg, seed,
                                                  field, remap, scale);
    return cudaGetLastError();
}

// ---- device-side bitwise compare of a device-layout field against an X-pitched host block ----
// Local planes [k0, k0 + nk) of `dev` against `blk` ([nk][Y][X]); counts differing cells and
// keeps the lowest global linear index (base + block index) of a difference.
__global__ void compare_field_kernel(const double* __restrict__ dev, int pitch, int off, int X,
                                     int Y, int k0, int nk, const double* __restrict__ blk,
                                     long long base, unsigned long long* count,
                                     unsigned long long* first) {
    const long long n = static_cast<long long>(nk) * Y * X;
    unsigned long long local = 0, lo = ~0ull;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(q % X);
        const long long r = q / X;
        const int j = static_cast<int>(r % Y);
        const int k = static_cast<int>(r / Y);
        const double a = dev[(static_cast<long long>(k0 + k) * Y + j) * pitch + off + i];
        if (__double_as_longlong(a) != __double_as_longlong(blk[q])) {
            ++local;
            lo = min(lo, static_cast<unsigned long long>(base + q));
        }
    }
    if (local) {
        atomicAdd(count, local);
        atomicMin(first, lo);
    }
}

cudaError_t launch_compare_field(const double* dev, int pitch, int off, int X, int Y, int k0,
                                 int nk, const double* blk, long long base,
                                 unsigned long long* count, unsigned long long* first,
                                 int sm_count, cudaStream_t stream) {
    compare_field_kernel<<<sm_count * 8, 256, 0, stream>>>(dev, pitch, off, X, Y, k0, nk, blk,
                                                           base, count, first);
    return cudaGetLastError();
}

// ---- row digest: FNV-1a (64-bit) of the bytes of each allocated row (k, j) of local planes
// [k0, k0 + nk), i.e. the X elements at device offset `off`, in host order. One thread per row;
// the host folds the row hashes (girih_gpu_row_digest). ----
__global__ void row_fnv_kernel(const double* __restrict__ dev, int pitch, int off, int X, int Y,
                               int k0, int nk, unsigned long long* __restrict__ out) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r >= static_cast<long long>(nk) * Y) return;
    const int k = static_cast<int>(r / Y), j = static_cast<int>(r % Y);
    const double* row = dev + (static_cast<long long>(k0 + k) * Y + j) * pitch + off;
    unsigned long long h = 0xCBF29CE484222325ull;
    for (int i = 0; i < X; ++i) {
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(row[i]));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            h ^= (b >> (8 * q)) & 0xFFull;
            h *= 0x100000001B3ull;
        }
    }
    out[r] = h;
}

cudaError_t launch_row_fnv(const double* dev, int pitch, int off, int X, int Y, int k0, int nk,
                           unsigned long long* out, cudaStream_t stream) {
    const long long rows = static_cast<long long>(nk) * Y;
    const int block = 128;
    row_fnv_kernel<<<static_cast<unsigned>((rows + block - 1) / block), block, 0, stream>>>(
        dev, pitch, off, X, Y, k0, nk, out);
    return cudaGetLastError();
}

// ---- ghost shell of a field: scatter a packed [plane][shell] block into the device layout ----
// Allocated planes [k0, k0 + nk) of a field whose interior is not needed (the input level t0-1
// of a Jacobi run: overwritten before any read): ghost planes in full, in the other planes the
// R ghost rows at each y end in full and, in every interior row, the R ghost cells left of the
// interior and the R ghost + pad cells right of it. One block per (plane, row).
__global__ void scatter_shell_kernel(double* dev, int pitch, int off, int X, int Y, int R, int nx,
                                     int ny, int nzg, int k0, const double* packed) {
    const int j = blockIdx.x, kk = blockIdx.y, k = k0 + kk;
    const long long S = 2LL * R * X + (long long)ny * (X - nx);  // interior-plane shell
    // packed offset of plane k: ghost planes before it are full planes
    const int gbefore = min(k0, R) + max(0, k0 - (R + nzg));       // ghost planes before k0
    const int ibefore = k0 - gbefore;                              // interior planes before k0
    long long base = 0;
    // planes of this chunk before k
    for (int q = k0; q < k; ++q) base += (q < R || q >= R + nzg) ? (long long)X * Y : S;
    base += (long long)gbefore * X * Y + (long long)ibefore * S;
    double* row = dev + ((long long)k * Y + j) * pitch + off;
    const bool gplane = k < R || k >= R + nzg;
    if (gplane || j < R || j >= R + ny) {
        const long long o = gplane ? base + (long long)j * X
                                   : base + (j < R ? (long long)j * X
                                                   : (long long)R * X + (long long)ny * (X - nx) +
                                                         (long long)(j - R - ny) * X);
        for (int i = threadIdx.x; i < X; i += blockDim.x) row[i] = packed[o + i];
    } else {
        const long long o = base + (long long)R * X + (long long)(j - R) * (X - nx);
        for (int i = threadIdx.x; i < X - nx; i += blockDim.x)
            row[i < R ? i : i + nx] = packed[o + i];
    }
}

cudaError_t launch_scatter_shell(double* dev, int pitch, int off, int X, int Y, int R, int nx,
                                 int ny, int nzg, int k0, int nk, const double* packed,
                                 cudaStream_t stream) {
    scatter_shell_kernel<<<dim3(Y, nk), 64, 0, stream>>>(dev, pitch, off, X, Y, R, nx, ny, nzg, k0,
                                                         packed);
    return cudaGetLastError();
}

// ---- FP64 rate probe: independent chains of DADD/DMUL (bitwise mode) or DFMA ----
template <int MODE>
__global__ void fp64_probe_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int n = 0; n < iters; ++n) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) {
                x0 = __dadd_rn(__dmul_rn(x0, a), b); x1 = __dadd_rn(__dmul_rn(x1, a), b);
                x2 = __dadd_rn(__dmul_rn(x2, a), b); x3 = __dadd_rn(__dmul_rn(x3, a), b);
                x4 = __dadd_rn(__dmul_rn(x4, a), b); x5 = __dadd_rn(__dmul_rn(x5, a), b);
                x6 = __dadd_rn(__dmul_rn(x6, a), b); x7 = __dadd_rn(__dmul_rn(x7, a), b);
            } else {
                x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b);
                x3 = __fma_rn(x3, a, b); x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b);
                x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
            }
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

cudaError_t launch_fp64_probe(int mode, double* out, int blocks, int threads, int iters,
                              cudaStream_t stream) {
    if (mode == 0)
        fp64_probe_kernel<0><<<blocks, threads, 0, stream>>>(out, iters, 0.999999, 1e-7);
    else
        fp64_probe_kernel<1><<<blocks, threads, 0, stream>>>(out, iters, 0.999999, 1e-7);
    return cudaGetLastError();
}

}  // namespace girih_gpu
