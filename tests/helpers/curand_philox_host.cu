// Test helper: exposes cuRAND's own Philox4x32-10 round function, compiled for the
// HOST (curand_philox4x32_x.h carries an explicit NV_IS_HOST path), as a C symbol.
// Used only to pin oracle/shuf_oracle.c's D1 against a library routine on any
// counter, including nonzero x1/x3 words the host generator API never reaches.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <stdint.h>

extern "C" void curand_ref_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out, uint64_t count) {
    for (uint64_t i = 0; i < count; i++) {
        uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
        uint2 k = make_uint2(key[2 * i], key[2 * i + 1]);
        uint4 r = curand_Philox4x32_10(c, k);
        out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
    }
}
