/* Host memory bandwidth probe (pageable e2e analysis): T threads
 * copy a 2 GiB buffer with streaming (non-temporal) stores; prints the copy
 * rate and the DRAM traffic it implies (read + write).
 *   gcc -O2 -mavx2 -pthread -o /tmp/host_bw tools/dbg/host_bw.c && /tmp/host_bw 16 */
#include <emmintrin.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char *src, *dst;
static size_t total;
static int nthr;

static void* work(void* arg) {
    const long t = (long)arg;
    const size_t per = total / nthr;
    char* d = dst + t * per;
    const char* s = src + t * per;
    for (size_t i = 0; i + 64 <= per; i += 64) {
        __m128i a = _mm_loadu_si128((const __m128i*)(s + i)), b = _mm_loadu_si128((const __m128i*)(s + i + 16)),
                c = _mm_loadu_si128((const __m128i*)(s + i + 32)), e = _mm_loadu_si128((const __m128i*)(s + i + 48));
        _mm_stream_si128((__m128i*)(d + i), a);
        _mm_stream_si128((__m128i*)(d + i + 16), b);
        _mm_stream_si128((__m128i*)(d + i + 32), c);
        _mm_stream_si128((__m128i*)(d + i + 48), e);
    }
    _mm_sfence();
    return NULL;
}

int main(int argc, char** argv) {
    nthr = argc > 1 ? atoi(argv[1]) : 16;
    total = (size_t)1 << 31;
    src = aligned_alloc(4096, total);
    dst = aligned_alloc(4096, total);
    memset(src, 1, total);
    memset(dst, 2, total);
    for (int rep = 0; rep < 3; ++rep) {
        pthread_t th[256];
        struct timespec t0, t1;
        clock_gettime(CLOCK_MONOTONIC, &t0);
        for (long t = 0; t < nthr; ++t) pthread_create(&th[t], NULL, work, (void*)t);
        for (int t = 0; t < nthr; ++t) pthread_join(th[t], NULL);
        clock_gettime(CLOCK_MONOTONIC, &t1);
        const double s = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
        printf("threads %d: copy %.1f GB/s, DRAM traffic %.1f GB/s\n", nthr, total / s / 1e9, 2 * total / s / 1e9);
    }
    return 0;
}
