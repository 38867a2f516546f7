// CPU prototype 2: plain Jacobi (entry_k <- exit_{k-1} of the previous round) for the exact
// PrevValue chain; reports rounds, recomputed elements, and per-chunk merge statistics.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static double EB = 1e-3, STEP = 2e-3; static int64_t R = 32768;
static inline float qs(float xf, double pred) {
    const double orig = xf; const double q = round((orig - pred) / STEP);
    if (fabs(q) < (double)R) { const float cand = (float)(pred + q * STEP);
        if (isfinite(cand) && fabs(orig - (double)cand) <= EB) return cand; }
    return xf; }
static double gauss(void) { double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0); return sqrt(-2 * log(u)) * cos(6.283185307179586 * v); }
int main(int argc, char** argv) {
    long P = atol(argv[1]); int L = atoi(argv[2]); int relu = atoi(argv[3]); int planes = atoi(argv[4]);
    int guess_mode = argc > 5 ? atoi(argv[5]) : 0;  // 0 ideal lattice, 1 warm-up spec of W=L elements
    if (argc > 6) { EB = atof(argv[6]); STEP = 2 * EB; }
    srand(777);
    float* x = malloc(4 * P); float* tr = malloc(4 * P);
    long nch = (P + L - 1) / L;
    float *a = malloc(4 * nch), *E = malloc(4 * nch), *pa = malloc(4*nch);
    double sum_rounds = 0; long max_rounds = 0, rec_elems = 0, conv = 0, tot_ch = 0;
    long hist[40] = {0};
    for (int p = 0; p < planes; ++p) {
        for (long i = 0; i < P; ++i) { double g = gauss(); x[i] = relu ? (g > 0 ? g : 0) : g; }
        float r = 0; for (long i = 0; i < P; ++i) { r = qs(x[i], i ? (double)r : 0.0); tr[i] = r; }
        for (long k = 0; k < nch; ++k) {
            long s = k * L;
            if (k == 0) a[k] = 0;
            else if (guess_mode == 0) a[k] = (float)(round((double)x[s - 1] / STEP) * STEP);
            else { // warm-up: spec chain over the previous L elements from the ideal guess there
                long w0 = s - L; float g = (w0 == 0) ? 0.0f : (float)(round((double)x[w0 - 1] / STEP) * STEP);
                for (long i = w0; i < s; ++i) g = qs(x[i], i ? (double)g : 0.0);
                a[k] = g; rec_elems += L; }
        }
        int rounds = 0;
        for (long k = 0; k < nch; ++k) pa[k] = NAN;
        for (;;) {
            ++rounds; int changed = 0;
            for (long k = 0; k < nch; ++k) {
                if (!(a[k] == pa[k] && !isnan(pa[k])) || (rounds == 1)) {
                    long s = k * L, e = s + L < P ? s + L : P; float r2 = a[k];
                    for (long i = s; i < e; ++i) r2 = qs(x[i], i ? (double)r2 : 0.0);
                    E[k] = r2; rec_elems += e - s; pa[k] = a[k];
                    if (rounds == 1) { tot_ch++; conv += (E[k] == tr[e - 1]); }
                }
            }
            for (long k = 1; k < nch; ++k) if (a[k] != E[k - 1]) { a[k] = E[k - 1]; changed = 1; }
            if (!changed) break;
        }
        if (E[nch - 1] != tr[P - 1]) { printf("MISMATCH\n"); return 1; }
        sum_rounds += rounds; if (rounds > max_rounds) max_rounds = rounds; hist[rounds < 39 ? rounds : 39]++;
    }
    printf("P=%ld L=%d relu=%d guess=%d eb=%g: rounds mean %.2f max %ld | work %.2fx | P(exit ok round1) %.3f\n", P, L, relu,
           guess_mode, EB, sum_rounds / planes, max_rounds, (double)rec_elems / ((double)P * planes), (double)conv / tot_ch);
}
