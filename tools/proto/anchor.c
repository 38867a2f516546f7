// CPU prototype 3: anchored speculation. Each chunk's speculative chain starts at the last
// "anchor" (element whose |x| lies in the top frequent binade, so the true-vs-spec offset is
// a multiple of the coarsest grid) within Wmax elements before the chunk start. Chunk entry
// offsets then come from a prefix sum of defects (translation). Measures how many chunks the
// translation prediction gets exactly right (symbols + exit), and the warm-up overhead.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static double EB = 1e-3, STEP = 2e-3; static int64_t R = 32768;
static inline uint32_t qs(float xf, double pred, float* out, double* pre) {
    const double orig = xf; const double q = round((orig - pred) / STEP);
    if (fabs(q) < (double)R) { double y = pred + q * STEP; const float cand = (float)y;
        if (isfinite(cand) && fabs(orig - (double)cand) <= EB) { *out = cand; *pre = y; return (uint32_t)((int64_t)q + R);} }
    *out = xf; *pre = NAN; return 0; }
static double gauss(void) { double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0); return sqrt(-2 * log(u)) * cos(6.283185307179586 * v); }
int main(int argc, char** argv) {
    long P = atol(argv[1]); int L = atoi(argv[2]); int relu = atoi(argv[3]); int planes = atoi(argv[4]);
    double A = atof(argv[5]); int Wmax = atoi(argv[6]); if (argc > 7) { EB = atof(argv[7]); STEP = 2 * EB; }
    srand(4242);
    float *x = malloc(4*P), *tr = malloc(4*P); uint32_t* tsym = malloc(4*P); double* tpre = malloc(8*P);
    long nch = (P + L - 1) / L;
    float* sstart = malloc(4*nch); float* send = malloc(4*nch); double* yend = malloc(8*nch);
    int* ok_sym = malloc(4*nch); double* D = malloc(8*nch);
    long tot = 0, bad_sym = 0, bad_exit = 0, bad_any = 0, warm = 0, noanchor = 0;
    for (int p = 0; p < planes; ++p) {
        for (long i = 0; i < P; ++i) { double g = gauss(); x[i] = relu ? (g > 0 ? g : 0) : g; }
        float r = 0; for (long i = 0; i < P; ++i) { double pre; tsym[i] = qs(x[i], i ? (double)r : 0.0, &r, &pre); tr[i] = r; tpre[i]=pre; }
        for (long k = 0; k < nch; ++k) {
            long s = k * L, e = s + L < P ? s + L : P;
            // find anchor
            long a = -1;
            if (k > 0) for (long i = s - 1; i >= 0 && i >= s - Wmax; --i) if (fabs(x[i]) >= A) { a = i; break; }
            float st; long from;
            if (k == 0) { st = 0; from = 0; }
            else if (a >= 0) { st = (float)(round((double)x[a] / STEP) * STEP); from = a + 1; }
            else { noanchor++; st = (float)(round((double)x[s-1] / STEP) * STEP); from = s; }
            warm += s - from;
            float rr = st; double pre = NAN, ylast = NAN; ok_sym[k] = 1;
            for (long i = from; i < e; ++i) {
                if (i == s) sstart[k] = rr;
                uint32_t q = qs(x[i], i ? (double)rr : 0.0, &rr, &pre);
                if (!isnan(pre) && (double)rr - pre != 0.0 ) {}
                if (x[i] != 0 || 1) { if (q && !(x[i]==0 && fabs(rr) < 1e-3)) ylast = pre; else if (q) ylast = pre; }
                if (i >= s && q != tsym[i]) ok_sym[k] = 0;
            }
            if (from == s && k == 0) sstart[k] = 0;
            send[k] = rr; yend[k] = ylast;
        }
        // scan: D_k = t_start_k - s_start_k predicted via D_k = D_{k-1} + (send_{k-1} - sstart_k)
        D[0] = 0;
        for (long k = 1; k < nch; ++k) {
            // predicted true exit of k-1
            double pe = (double)send[k-1] + D[k-1];
            D[k] = pe - (double)sstart[k];
        }
        for (long k = 0; k < nch; ++k) {
            long e = (k + 1) * L < P ? (k + 1) * L : P;
            double tstart = (k == 0) ? 0.0 : (double)tr[k * L - 1];
            int start_ok = (k == 0) || ((double)sstart[k] + D[k] == tstart);
            // predicted exit: translation
            float pred_exit = (float)((double)send[k] + D[k]);
            int exit_ok = pred_exit == tr[e - 1];
            tot++; bad_sym += !ok_sym[k]; bad_exit += !exit_ok; bad_any += !(ok_sym[k] && exit_ok && start_ok);
        }
    }
    printf("P=%ld L=%d relu=%d A=%g W=%d eb=%g: chunks %ld  bad_sym %.4f bad_exit %.4f bad_any %.4f  warmup %.2f noanchor %.4f\n",
        P, L, relu, A, Wmax, EB, tot, (double)bad_sym/tot, (double)bad_exit/tot, (double)bad_any/tot, (double)warm/(P*(double)planes), (double)noanchor/tot);
}
