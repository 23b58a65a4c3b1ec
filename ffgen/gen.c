/* gen.c -- the same counter-based generator as ffgen/__init__.py, in C with
 * OpenMP, for the large host inputs the bench's CPU checks need (the numpy
 * version generates ~27 M elements/s).  Holds none of the method's
 * arithmetic: splitmix64's output function and a final "mod p" only.
 *   v[i] = (mix64(key + (i + 1) * GAMMA) >> 11) mod p,  i = start .. start+count-1 */
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void ffgen_uniform_flat(uint32_t p, uint64_t key, int64_t start, int64_t count, int32_t *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t z = key + (uint64_t)(start + i + 1) * 0x9E3779B97F4A7C15ULL;
        out[i] = (int32_t)((mix64(z) >> 11) % p);
    }
}

/* Threads for the loop above (0: leave the OpenMP default); torchrun sets
 * OMP_NUM_THREADS=1 for every rank, which the bench's per-rank checks override. */
void ffgen_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
