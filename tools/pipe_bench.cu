// pipe_bench.cu — issue-rate microbenchmarks for the int pipes of sm_100a (dev tool):
// LOP3 alone, IMAD.WIDE.U32 alone, and interleaved mixes, to see whether FMA-pipe integer
// multiply-adds can run beside the LOP3 stream of the Toeplitz kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NL, int NM>
__global__ void __launch_bounds__(256) k_mix(uint32_t iters, uint32_t* out, uint32_t mulv) {
    uint32_t a[16];
    unsigned long long m[8];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = (threadIdx.x + 1) * 0x9E3779B9u + j * 0x85EBCA6Bu;
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = (threadIdx.x + j) * 0x12345ull;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < NL; ++j) a[j & 15] ^= a[(j + 3) & 15] & a[(j + 7) & 15];
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                unsigned long long d;
                asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a[(j + 5) & 15]), "r"(mulv), "l"(m[j & 7]));
                m[j & 7] = d;
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) x ^= a[j];
#pragma unroll
    for (int j = 0; j < 8; ++j) x ^= (uint32_t)m[j] ^ (uint32_t)(m[j] >> 32);
    if (x == 0x12345678u) out[blockIdx.x] = x;
}

template <int NL, int NM>
void run(const char* name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mix<NL, NM>, 256, 0);
    const int grid = sms * per;
    uint32_t* out;
    cudaMalloc(&out, grid * 4);
    const uint32_t iters = 4000;
    k_mix<NL, NM><<<grid, 256>>>(200, out, 0x10001u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mix<NL, NM><<<grid, 256>>>(iters, out, 0x10001u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double warps = (double)grid * 8 * iters * 8;  // warp-iterations of the r loop
    const double cyc = ms * 1e-3 * 1.965e9;              // assume boost clock
    printf("%-12s occ=%d  LOP3/clk/SM=%.2f warp-instr  IMADW/clk/SM=%.2f warp-instr  ms=%.2f\n",
           name, per, warps * NL / cyc / sms, warps * NM / cyc / sms, ms);
    cudaFree(out);
}

int main() {
    run<16, 0>("lop3");
    run<0, 8>("imadw");
    run<16, 2>("16L:2M");
    run<16, 4>("16L:4M");
    run<16, 8>("16L:8M");
    run<8, 8>("8L:8M");
    return 0;
}
