// Host side of the grid solvers: shape/shared-memory sizing and launches of
// redrec_kernel (redrec.cu) and bird_kernel (bird.cu).

#include <algorithm>

#include "grid_common.cuh"

namespace rb {

__global__ void redrec_kernel(GridParams p);
__global__ void bird_kernel(GridParams p);

bool grid_shape(int W, int H, int k, int nwarps, GridShape &s) {
    if (W <= 0 || H <= 0 || W > 1024 || H > 1024) return false;
    s.W = W;
    s.H = H;
    s.k = k;
    s.wpd = (H + 63) / 64;
    const int need = (H + 31) / 32;
    s.B = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
    s.LK = k + 2;
    const int ylo = (H - k) / 2, yhi = ylo + k - 1;
    const int lo = H - 1 - yhi, hi = H - 1 - ylo;
    s.LT = (int)align_up(lo + W - 1 + 64, 64);
    s.LB = (int)align_up((H - 1 - hi) + W - 1 + 64, 64);
    s.nchunk = (2 * W - 1 + 31) / 32;
    s.nwarps = nwarps;
    GridSmem o;
    grid_smem_layout(s, o);
    s.smem_bytes = o.total;
    return s.smem_bytes <= 227 * 1024;
}

size_t grid_snap_words(const GridShape &s) { return (size_t)2 * s.W * s.wpd; }

cudaError_t launch_grid_solver(int solver, const GridParams &p, int grid, cudaStream_t stream) {
    const int threads = 32 * p.shape.nwarps;
    void (*kern)(GridParams) = solver == 0 ? redrec_kernel : bird_kernel;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.shape.smem_bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, p.shape.smem_bytes, stream>>>(p);
    return cudaGetLastError();
}

int grid_occupancy(int solver, const GridShape &s) {
    int nb = 0;
    void (*kern)(GridParams) = solver == 0 ? redrec_kernel : bird_kernel;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.smem_bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * s.nwarps, s.smem_bytes);
    return nb;
}

}  // namespace rb
