// Shared-memory access-pattern microbenchmark for the ranking / placement /
// Fisher-Yates design choices.  Every kernel runs NT threads per
// CTA, `ctas_per_sm` CTAs per SM, and issues ITER x 16 shared-memory warp
// instructions of one kind per warp; the host reports SM-cycles per warp
// instruction (time x clock x #SM / total warp instructions).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_smem tools/mb_smem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e) {                                                                  \
            printf("err %s line %d\n", cudaGetErrorString(e), __LINE__);          \
            return 1;                                                             \
        }                                                                         \
    } while (0)

constexpr int ITER = 256;
constexpr uint32_t WORDS = 16384;  // 64 KiB table

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// mode: 0 LDS contiguous, 1 LDS random (64 KiB), 2 STS random, 3 ATOMS random
// in a per-warp 128-word table (ranking), 4 ATOMS random (64 KiB), 5 RED (no
// return) per-warp table, 6 LDS random u8, 7 match_any 8-bit, 8 ballot x 8,
// 9 LDS random restricted to the lane's own bank, 10 LDS+STS swap pairs random
// (FY-like, 4 accesses), 11 STS random u8
template <int MODE>
__global__ void k_mb(uint32_t* out) {
    extern __shared__ uint32_t sm[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t i = tid; i < WORDS; i += blockDim.x) sm[i] = i;
    __syncthreads();
    uint32_t off[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t h = hash32(tid * 16 + j + blockIdx.x * 7919u);
        if (MODE == 0) off[j] = (warp * 32 * 16 + j * 32 + lane) & (WORDS - 1);
        else if (MODE == 3 || MODE == 5) off[j] = (WORDS - 2048) + (warp & 15) * 128 + (h & 127);
        else if (MODE == 7 || MODE == 8) off[j] = h & 255;
        else if (MODE == 9) off[j] = ((h & 511) << 5) | lane;
        else if (MODE == 6 || MODE == 11) off[j] = h & (WORDS * 4 - 1);
        else off[j] = h & (WORDS - 1);
    }
    uint32_t acc = 0;
    unsigned char* smb = reinterpret_cast<unsigned char*>(sm);
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t o = off[j] ^ (it & 1);
            if (MODE == 0 || MODE == 1 || MODE == 9) acc += sm[MODE == 0 ? off[j] : o];
            else if (MODE == 2) sm[o] = acc + j;
            else if (MODE == 3 || MODE == 4) acc += atomicAdd(&sm[off[j]], 1u);
            else if (MODE == 5) atomicAdd(&sm[off[j]], 1u);
            else if (MODE == 6) acc += smb[o];
            else if (MODE == 11) smb[o] = (unsigned char)(acc + j);
            else if (MODE == 7) acc += __match_any_sync(0xFFFFFFFFu, off[j] ^ (acc & 1));
            else if (MODE == 8) {
                uint32_t m = 0xFFFFFFFFu;
                const uint32_t b = off[j] ^ (acc & 1);
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const uint32_t bb = __ballot_sync(0xFFFFFFFFu, (b >> x) & 1);
                    m &= ((b >> x) & 1) ? bb : ~bb;
                }
                acc += m;
            } else if (MODE == 10) {
                const uint32_t a = off[j], b2 = hash32(off[j] + acc) & (WORDS - 1);
                const uint32_t x = sm[a], y = sm[b2];
                sm[a] = y;
                sm[b2] = x + 1;
                acc += x;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
static int run(const char* name, int nt, int cps, int sms, int clk_khz, uint32_t* d) {
    const int smem = WORDS * 4;
    CK(cudaFuncSetAttribute(k_mb<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = sms * cps;
    k_mb<MODE><<<grid, nt, smem>>>(d);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_mb<MODE><<<grid, nt, smem>>>(d);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr_per_sm = (double)reps * cps * (nt / 32) * ITER * 16;
    const double cyc = ms * 1e-3 * clk_khz * 1e3;
    printf("%-28s nt=%4d cps=%d  %.2f SM-cycles per warp-instruction\n", name, nt, cps, cyc / warp_instr_per_sm);
    return 0;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d clock %d kHz\n", sms, clk);
    uint32_t* d;
    CK(cudaMalloc(&d, 64));
    for (int cfg = 0; cfg < 2; ++cfg) {
        const int nt = cfg ? 512 : 1024, cps = cfg ? 2 : 1;
        run<0>("LDS contiguous", nt, cps, sms, clk, d);
        run<1>("LDS random", nt, cps, sms, clk, d);
        run<9>("LDS random own-bank", nt, cps, sms, clk, d);
        run<6>("LDS random u8", nt, cps, sms, clk, d);
        run<2>("STS random", nt, cps, sms, clk, d);
        run<11>("STS random u8", nt, cps, sms, clk, d);
        run<3>("ATOMS rand per-warp 128w", nt, cps, sms, clk, d);
        run<4>("ATOMS rand 64KiB", nt, cps, sms, clk, d);
        run<5>("RED per-warp 128w", nt, cps, sms, clk, d);
        run<7>("match_any 8-bit", nt, cps, sms, clk, d);
        run<8>("ballot x8 match", nt, cps, sms, clk, d);
        run<10>("FY swap (2 LDS+2 STS)", nt, cps, sms, clk, d);
    }
    return 0;
}
