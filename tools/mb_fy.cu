// Microbenchmark of the Fisher-Yates leaf chain: NT threads
// per CTA each run Fig. 1 on their own 64-element leaf held in shared memory,
// with precomputed partners, in several layouts/formulations; reports
// SM-cycles per item of 256 leaves (the HOT finish's unit of work).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_fy tools/mb_fy.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 64;     // leaf length
constexpr int REPS = 64;  // items per CTA

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// MODE 0: column layout (leaf of thread t: col[i*NT + t]), pull formulation,
//         final values to a contiguous out buffer, pipelined depth 1.
// MODE 1: contiguous leaf, in-place swaps, pipelined depth 1.
// MODE 2: column layout, in place, plain (no pipelining).
// MODE 3: column layout, in place, unrolled x4 (partner words per thread contiguous).
// MODE 4: column layout, in place, unrolled x4, partner words interleaved (conflict-free).
// MODE 5: contiguous leaf, in place, unrolled x4, partner words interleaved.
// MODE 6: column layout, pull to a contiguous out buffer, unrolled x4, interleaved partners.
template <int MODE, int NT>
__global__ void __launch_bounds__(NT, 1) k_fy(uint32_t* sink) {
    extern __shared__ uint32_t sm[];
    constexpr int NB = (MODE == 0 || MODE == 6) ? 2 : 1;  // word buffers of NT*M
    uint32_t* col = sm;                          // NT*M words
    uint32_t* out = (MODE == 0 || MODE == 6) ? sm + NT * M : sm;
    unsigned char* jb = (unsigned char*)(sm + NB * NT * M);  // NT*M bytes
    const uint32_t t = threadIdx.x;
    for (uint32_t i = t; i < NT * M; i += NT) {
        col[i] = i;
        const uint32_t leaf = i / M, step = i % M;
        jb[i] = (unsigned char)(step ? hash32(i * 7 + blockIdx.x) % (step + 1) : 0);
    }
    __syncthreads();
    const uint32_t* jw = (const uint32_t*)(jb + t * M);
    uint32_t acc = 0;
    for (int rep = 0; rep < REPS; ++rep) {
        if (MODE == 0) {
            uint32_t* c = col + t;
            uint32_t* o = out + t * M;
            uint32_t i = M - 1;
            uint32_t jc = (jw[i >> 2] >> ((i & 3) * 8)) & 0xFF;
            uint32_t x = c[i * NT], y = c[jc * NT];
            for (; i >= 2; --i) {
                const uint32_t jn = (jw[(i - 1) >> 2] >> (((i - 1) & 3) * 8)) & 0xFF;
                uint32_t xn = c[(i - 1) * NT], yn = c[jn * NT];
                c[jc * NT] = x;
                o[i] = y;
                if (jc == i - 1) xn = x;
                if (jn == jc) yn = x;
                x = xn;
                y = yn;
                jc = jn;
            }
            c[jc * NT] = x;
            o[1] = y;
            o[0] = c[0];
            acc += o[rep & 63];
        } else if (MODE == 1) {
            uint32_t* A = out + t * M;
            uint32_t i = M - 1;
            uint32_t jc = (jw[i >> 2] >> ((i & 3) * 8)) & 0xFF;
            uint32_t x = A[i], y = A[jc];
            for (; i >= 2; --i) {
                const uint32_t jn = (jw[(i - 1) >> 2] >> (((i - 1) & 3) * 8)) & 0xFF;
                uint32_t xn = A[i - 1], yn = A[jn];
                A[jc] = x;
                A[i] = y;
                if (jc == i - 1) xn = x;
                if (jn == jc) yn = x;
                x = xn;
                y = yn;
                jc = jn;
            }
            A[jc] = x;
            A[1] = y;
            acc += A[rep & 63];
        } else if (MODE == 2) {
            uint32_t* c = col + t;
            for (uint32_t i = M - 1; i >= 1; --i) {
                const uint32_t j = (jw[i >> 2] >> ((i & 3) * 8)) & 0xFF;
                const uint32_t x = c[i * NT], y = c[j * NT];
                c[j * NT] = x;
                c[i * NT] = y;
            }
            acc += c[(rep & 63) * NT];
        } else if (MODE == 4 || MODE == 5 || MODE == 6) {
            const uint32_t* jwi = (const uint32_t*)jb;  // word w of thread t at jwi[w*NT + t]
            uint32_t* c = MODE == 5 ? out + t * M : col + t;
            constexpr int S = MODE == 5 ? 1 : NT;
            uint32_t* o = out + t * M;
            uint32_t* ci = c + (M - 1) * S;
            for (int w = (M / 4) - 1; w >= 0; --w) {
                const uint32_t pk = jwi[w * NT + t];
#pragma unroll
                for (int q = 3; q >= 0; --q) {
                    if (w == 0 && q == 0) break;
                    const uint32_t j = (pk >> (q * 8)) & 0xFF;
                    uint32_t* cj = c + j * S;
                    const uint32_t x = *ci, y = *cj;
                    *cj = x;
                    if (MODE == 6) o[w * 4 + q] = y;
                    else *ci = y;
                    ci -= S;
                }
            }
            if (MODE == 6) o[0] = c[0];
            acc += MODE == 6 ? o[rep & 63] : c[(rep & 63) * S];
        } else {
            // partners unpacked 4 at a time, explicit unroll, pointer walking
            uint32_t* c = col + t;
            uint32_t* ci = c + (M - 1) * NT;
            for (int w = (M / 4) - 1; w >= 0; --w) {
                const uint32_t pk = jw[w];
#pragma unroll
                for (int q = 3; q >= 0; --q) {
                    if (w == 0 && q == 0) break;
                    const uint32_t j = (pk >> (q * 8)) & 0xFF;
                    uint32_t* cj = c + j * NT;
                    const uint32_t x = *ci, y = *cj;
                    *cj = x;
                    *ci = y;
                    ci -= NT;
                }
            }
            acc += c[(rep & 63) * NT];
        }
    }
    if (acc == 0x9876543u) sink[0] = acc;
}

template <int MODE, int NT>
static void run(const char* name, int sms, int clk_khz, uint32_t* d) {
    const int smem = NT * M * 4 * ((MODE == 0 || MODE == 6) ? 2 : 1) + NT * M;
    cudaFuncSetAttribute(k_fy<MODE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_fy<MODE, NT><<<sms, NT, smem>>>(d);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_fy<MODE, NT><<<sms, NT, smem>>>(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const cudaError_t e = cudaGetLastError();
    const double cyc = ms * 1e-3 * clk_khz * 1e3 / REPS;  // per rep (NT leaves of 64)
    printf("%-34s NT=%4d: %8.0f cycles per %d leaves -> %7.0f cycles per 256 leaves  %s\n", name, NT, cyc, NT,
           cyc * 256.0 / NT, e ? cudaGetErrorString(e) : "");
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* d;
    cudaMalloc(&d, 64);
    run<3, 256>("column in-place unrolled", sms, clk, d);
    run<4, 256>("column in-place unr, jw interleaved", sms, clk, d);
    run<5, 256>("contig in-place unr, jw interleaved", sms, clk, d);
    run<6, 256>("column pull unr, jw interleaved", sms, clk, d);
    run<4, 512>("column in-place unr, jw interleaved", sms, clk, d);
    run<5, 512>("contig in-place unr, jw interleaved", sms, clk, d);
    run<5, 1024>("contig in-place unr, jw interleaved", sms, clk, d);
    return 0;
}
