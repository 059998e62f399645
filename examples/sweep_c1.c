/* Minimal C client of the sb200 C ABI (include/sb200.h): the C1 stencil
 * (1D 3-point, weights 0.25/0.5/0.25) over a seeded line, T steps on the GPU in
 * EXACT arithmetic, checked against a plain C loop of the reference's scalar
 * step (acc = 0; acc += w*x per canonical offset, kernels.py:103-108).
 *
 *   gcc -O2 -ffp-contract=off -I include examples/sweep_c1.c \
 *       -L paper_2103_08825_b200/lib -lsb200 -Wl,-rpath,$PWD/paper_2103_08825_b200/lib -o sweep_c1
 *   ./sweep_c1 [n] [T]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sb200.h"

static int check(int rc, const char *what) {
    if (rc != SB_OK) fprintf(stderr, "%s failed (%d): %s\n", what, rc, sb_last_error());
    return rc;
}

int main(int argc, char **argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 100003;
    const int64_t T = argc > 2 ? atoll(argv[2]) : 37;
    const int32_t offsets[3] = {-1, 0, 1};
    const double weights[3] = {0.25, 0.5, 0.25};
    sb_problem p;
    memset(&p, 0, sizeof p);
    p.d = 1;
    p.r = 1;
    p.shape = SB_STAR;
    p.nw = 3;
    p.offsets = offsets;
    p.weights = weights;
    p.dims[0] = n;
    p.dtype = SB_F64;
    p.arith = SB_ARITH_EXACT;
    p.k = 8;
    p.kernel = SB_KERNEL_AUTO;

    const int64_t len = n + 2;                      /* halo-inclusive box */
    double *box = malloc(len * sizeof(double)), *out = malloc(len * sizeof(double));
    double *a = malloc(len * sizeof(double)), *b = malloc(len * sizeof(double));
    uint64_t s = 12345;
    for (int64_t i = 0; i < len; i++) {              /* xorshift: any seeded input will do */
        s ^= s << 13, s ^= s >> 7, s ^= s << 17;
        box[i] = (double)(s >> 11) / 9007199254740992.0;
    }
    sb_plan *plan = NULL;
    if (check(sb_plan_create(&plan, &p), "sb_plan_create")) return 2;
    sb_timing t;
    if (check(sb_upload(plan, box, len * sizeof(double)), "sb_upload") ||
        check(sb_run(plan, T, &t), "sb_run") || check(sb_download(plan, out, len * sizeof(double)), "sb_download"))
        return 2;
    sb_plan_destroy(plan);

    memcpy(a, box, len * sizeof(double));            /* reference: T scalar steps, fixed halo */
    memcpy(b, box, len * sizeof(double));
    for (int64_t step = 0; step < T; step++) {
        for (int64_t i = 1; i <= n; i++) {
            double acc = 0.0;
            for (int o = 0; o < 3; o++) acc = acc + weights[o] * a[i + offsets[o]];
            b[i] = acc;
        }
        double *tmp = a; a = b; b = tmp;
    }
    const int same = memcmp(a, out, len * sizeof(double)) == 0;
    printf("%s: %lld points x %lld steps, %s, %lld launches, %.3f ms on the device\n",
           same ? "bit-identical" : "MISMATCH", (long long)n, (long long)T, t.kernel_name,
           (long long)t.launches, t.device_ms);
    free(box), free(out), free(a), free(b);
    return same ? 0 : 1;
}
