// diag.cu — roofline denominator: measured LOP3 issue rate of this GPU.
//
// MEASURED_PEAKS.json holds only HBM and bf16 tensor peaks, so the integer-ALU peak the
// hash kernel is judged against is measured live: every SM runs independent
// acc ^= a & b chains (each one LOP3.LUT 0x78, the hash kernel's inner instruction) at
// full occupancy, timed with CUDA events.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssbh_cuda.h"

namespace {

__global__ void __launch_bounds__(256) k_lop3_peak(uint32_t iters, uint32_t* out) {
    uint32_t a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = (threadIdx.x + 1) * 0x9E3779B9u + j * 0x85EBCA6Bu;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] ^= a[(j + 3) & 15] & a[(j + 7) & 15];
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) x ^= a[j];
    if (x == 0x12345678u) out[blockIdx.x] = x;  // keep the chains live
}

}  // namespace

extern "C" ssbh_status ssbh_measure_lop3_peak(uint32_t iters, double* lop3_per_s, double* ms_out) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SSBH_NO_DEVICE;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lop3_peak, 256, 0);
    const int grid = sms * (per_sm > 0 ? per_sm : 1);
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, grid * 4) != cudaSuccess) return SSBH_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lop3_peak<<<grid, 256>>>(iters / 8 + 1, out);  // warm-up / clock ramp
    cudaEventRecord(e0);
    k_lop3_peak<<<grid, 256>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return SSBH_CUDA;
    const double ops = (double)grid * 256.0 * iters * 8.0 * 16.0;
    if (lop3_per_s) *lop3_per_s = ops / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return SSBH_OK;
}
