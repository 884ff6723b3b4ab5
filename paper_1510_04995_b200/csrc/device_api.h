// device_api.h -- host-callable launchers for the helper kernels (init_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace girih_gpu {

cudaError_t launch_init_field(double* buf, int pitch, int off, int X, int Y, int Zloc, int zoff,
                              int Zg, uint64_t seed, int field, int remap, double scale,
                              cudaStream_t stream);

// bitwise compare of local planes [k0, k0+nk) of a device-layout field with an X-pitched block
cudaError_t launch_compare_field(const double* dev, int pitch, int off, int X, int Y, int k0,
                                 int nk, const double* blk, long long base,
                                 unsigned long long* count, unsigned long long* first,
                                 int sm_count, cudaStream_t stream);

// per-row FNV-1a hashes of local planes [k0, k0+nk) (rows in k, j order) into out[nk * Y]
cudaError_t launch_row_fnv(const double* dev, int pitch, int off, int X, int Y, int k0, int nk,
                           unsigned long long* out, cudaStream_t stream);

// ghost shell (ghost planes, ghost rows, ghost/pad columns) of allocated planes [k0, k0+nk) from
// a packed host-order block (see init_kernels.cu)
cudaError_t launch_scatter_shell(double* dev, int pitch, int off, int X, int Y, int R, int nx,
                                 int ny, int nzg, int k0, int nk, const double* packed,
                                 cudaStream_t stream);

// mode 0: separate DMUL+DADD chains (2 ops per step), mode 1: DFMA chains (2 flops per step)
cudaError_t launch_fp64_probe(int mode, double* out, int blocks, int threads, int iters,
                              cudaStream_t stream);

}  // namespace girih_gpu
