// host int64 -> int32 narrowing bandwidth (OpenMP), to size the upload pipeline
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static double now(void) { return omp_get_wtime(); }
int main(int argc, char** argv) {
    const size_t m = argc > 1 ? strtoull(argv[1], 0, 10) : 132504180ull;
    int64_t* in = (int64_t*)malloc(m * 8);
    int32_t* out = (int32_t*)malloc(m * 4);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < m; ++i) { in[i] = (int64_t)(i * 2654435761u % 4194304u); out[i] = 0; }
    for (int th = 1; th <= omp_get_max_threads(); th *= 2) {
        omp_set_num_threads(th);
        double best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            const double t = now();
#pragma omp parallel for schedule(static)
            for (size_t i = 0; i < m; ++i) out[i] = (int32_t)in[i];
            const double dt = now() - t;
            if (dt < best) best = dt;
        }
        printf("threads %d: %.2f ms, read %.1f GB/s\n", th, best * 1e3, m * 8 / best / 1e9);
    }
    double t = now();
    memcpy(out, in, m * 4);
    printf("memcpy %zu MB single thread: %.2f ms\n", m * 4 >> 20, (now() - t) * 1e3);
    return out[m / 2] == 7;
}
