// CPU prototype: chunk-parallel exact PrevValue chain via Jacobi rounds with translation
// prediction. Measures rounds / recomputations to reach bit-exact consistency.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double EB = 1e-3, STEP = 2e-3; static int64_t R = 32768;

static inline uint32_t qstep(float xf, double pred, float* val) {
    const double orig = xf;
    const double q = round((orig - pred) / STEP);
    if (fabs(q) < (double)R) {
        const float cand = (float)(pred + q * STEP);
        if (isfinite(cand) && fabs(orig - (double)cand) <= EB) { *val = cand; return (uint32_t)((int64_t)q + R); }
    }
    *val = xf; return 0;
}
// runs chunk [s,e) of a plane (plane start at ps) from entry a; returns exit
static float run_chunk(const float* x, long s, long e, long ps, float a, uint32_t* sym) {
    float r = a;
    for (long i = s; i < e; ++i) {
        double pred = (i == ps) ? 0.0 : (double)r;
        float v; uint32_t q = qstep(x[i], pred, &v);
        if (sym) sym[i] = q;
        r = v;
    }
    return r;
}
static double gauss(void) { double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0); return sqrt(-2 * log(u)) * cos(6.283185307179586 * v); }

int mode_guess = 0; // 0 ideal lattice of x[s-1]

// process one plane of P elements with chunk length L; returns rounds; adds recomputes
static int plane(const float* x, long P, int L, long* recompute, long* maxr, int* bad) {
    long nch = (P + L - 1) / L;
    float* a = malloc(sizeof(float) * nch); float* E = malloc(sizeof(float) * nch);
    int* dirty = malloc(sizeof(int) * nch);
    for (long k = 0; k < nch; ++k) {
        long s = k * L;
        if (k == 0) a[k] = 0.0f;
        else { double K = round((double)x[s - 1] / STEP); a[k] = (float)(K * STEP); }
        dirty[k] = 1;
    }
    int rounds = 0;
    for (;;) {
        ++rounds;
        for (long k = 0; k < nch; ++k) if (dirty[k]) {
            long s = k * L, e = s + L < P ? s + L : P;
            E[k] = run_chunk(x, s, e, 0, a[k], NULL); (*recompute)++; dirty[k] = 0;
        }
        // consistency + defects
        double D = 0; int any = 0;
        for (long k = 1; k < nch; ++k) {
            double d = (double)E[k - 1] - (double)a[k];
            int cons = (E[k - 1] == a[k]) && !(signbit(E[k-1]) != signbit(a[k]));
            if (!cons) any = 1;
            D += cons ? 0.0 : d;
            if (D != 0.0) {
                float na = (float)((double)a[k] + D);
                if (!cons && na != E[k-1] && k>0) {}
                if (na != a[k]) { a[k] = na; dirty[k] = 1; }
                else if (!cons) { a[k] = E[k-1]; dirty[k] = 1; }
            } else if (!cons) { a[k] = E[k - 1]; dirty[k] = 1; }
        }
        if (!any) break;
        if (rounds > 200) { *bad = 1; break; }
    }
    // verify vs serial
    float es = run_chunk(x, 0, P, 0, 0.0f, NULL);
    if (es != E[nch - 1]) *bad = 2;
    if (rounds > *maxr) *maxr = rounds;
    free(a); free(E); free(dirty);
    return rounds;
}

int main(int argc, char** argv) {
    long P = argc > 1 ? atol(argv[1]) : 3136; int L = argc > 2 ? atoi(argv[2]) : 32;
    int relu = argc > 3 ? atoi(argv[3]) : 1; int planes = argc > 4 ? atoi(argv[4]) : 200;
    if (argc > 5) { EB = atof(argv[5]); STEP = 2 * EB; }
    srand(12345);
    float* x = malloc(sizeof(float) * P);
    long rec = 0, maxr = 0; double sumr = 0; int bad = 0; long hist[10] = {0};
    for (int p = 0; p < planes; ++p) {
        for (long i = 0; i < P; ++i) { double g = gauss(); x[i] = (float)(relu ? (g > 0 ? g : 0) : g); }
        int r = plane(x, P, L, &rec, &maxr, &bad);
        sumr += r; hist[r < 9 ? r : 9]++;
    }
    long nch = (P + L - 1) / L;
    printf("P=%ld L=%d relu=%d eb=%g: mean rounds %.2f max %ld, recompute/chunk %.2f bad=%d  hist:", P, L, relu, EB,
           sumr / planes, maxr, (double)rec / (planes * nch), bad);
    for (int i = 1; i < 10; ++i) printf(" %ld", hist[i]);
    printf("\n");
}
