/* CPU prototype of the "lattice chain": an exact, shorter-latency form of the reference
 * PrevValue recurrence (ref src/codec.cpp:76-104), validated bit for bit against the plain
 * reference step on many distributions before it goes into the CUDA kernels.
 *
 *   gcc -O2 -ffp-contract=off -o /tmp/dchain tools/proto/dchain.c -lm && /tmp/dchain
 *
 * Idea. With K = round(x/s) (s = 2 eb) and A = RN64(K s), the reference output is
 *   r = RN32(RN64(pred + RN64(q s))),  q = K - Kp,  pred = Ap + D  (D = drift, tiny),
 * i.e. r = RN32(A + D + err) with |err| <= ~2^-51 (|Ap| + |A|). With F = RN32(A) in binade
 * b (ulp u) and e = A - F, r = F + u * rint((e + D) / u) whenever (e + D)/u is not near a
 * half-integer and the result stays inside binade b. Everything but D is a function of x
 * alone, so the dependent chain per element is: t = fma(r, 1/u, H); m = rint(t);
 * r' = fma(m, u, F) -- four FP64 operations instead of the reference's ~12. Decisions
 * are certified by margins (|D| far from the decision / acceptance edges); anything else
 * (ties, binade edges, escapes, huge or tiny values) takes the reference step.
 * K = 0 elements (ReLU zeros): r = RN32(D) exactly.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double eb, s, inv_s, Rd;
    long long R;
} P;

static uint32_t ref_step(float xf, double pred, const P* p, double* r) {
    const double orig = xf;
    const double q = round((orig - pred) / p->s);
    if (fabs(q) < p->Rd) {
        const float cand = (float)(pred + q * p->s);
        if (isfinite(cand) && fabs(orig - (double)cand) <= p->eb) {
            *r = cand;
            return (uint32_t)((long long)q + p->R);
        }
    }
    *r = orig;
    return 0;
}

static double pow2i(int k) { return ldexp(1.0, k); }

/* the lattice chain over one plane; returns number of slow steps. The lattice is
 * {lam + K s}: lam = 0 at the plane start (pred = 0) and the value of the last escape after
 * one (the reference then predicts from the verbatim value, src/codec.cpp:96-99). */
static long g_rebase = 0;
static int g_mode = 1; /* 1: predicted-q chain, 0: lattice-output chain */ /* > 0: restart the lattice at the current state every g_rebase
                             elements (a chunk entry from a recorded state, as the replay does) */
static long chain_plane(const float* x, long n, const P* p, uint32_t* sym, float* out) {
    double r = 0.0;        /* pred: the previous output, exactly */
    double lam = 0.0;      /* lattice origin (a float) */
    long long Kp = 0;      /* lattice index of the previous output */
    double Ap = 0.0;       /* RN64(lam + RN64(Kp * s)) */
    long slow = 0;
    for (long i = 0; i < n; ++i) {
        if (g_rebase && i && i % g_rebase == 0) { /* chunk entry: lattice through the state */
            lam = r;
            Kp = 0;
            Ap = r;
        }
        const float xf = x[i];
        const double xd = xf;
        int fast = 0;
        double rn = 0.0;
        long long K = 0;
        uint32_t sy = 0;
        double A = 0.0;
        if (fabs(xd) < 0x1p100 && p->s > 0x1p-100) {
            const double tK = (xd - lam) * p->inv_s; /* xd - lam exact (two floats) */
            K = (long long)nearbyint(tK);
            const double Kd = (double)K;
            const double f = tK - Kd;
            const long long q = K - Kp;
            const double D = r - Ap; /* exact (Sterbenz) */
            const double slack1 = p->s * 0x1p-48 * (fabs(tK) + fabs((double)q) + 2.0) +
                                  0x1p-49 * (fabs(Ap) + fabs(lam));
            const double mdec = p->s * (0.5 - fabs(f)) - slack1;
            A = lam + Kd * p->s;
            if (llabs(q) < p->R && fabs(D) < mdec) {
                if (K == 0 && lam == 0.0) {
                    rn = (double)(float)D;
                    if (fabs(xd - rn) <= p->eb) fast = 1;
                } else {
                    const float F = (float)A;
                    const double Fd = F;
                    if (isfinite(F) && fabs(Fd) >= 0x1p-120 && A != 0.0) {
                        int b;
                        frexp(fabs(Fd), &b); /* |F| in [2^(b-1), 2^b) */
                        const double lo = pow2i(b - 1), hi = pow2i(b);
                        const double u = pow2i(b - 1 - 23), inv_u = pow2i(24 - b);
                        const double e = A - Fd;             /* exact */
                        const double H = (e - Ap) * inv_u;   /* rounded: covered by tie_eps */
                        const double t = fma(r, inv_u, H);
                        const double m = nearbyint(t);
                        const double tie_eps =
                            0x1p-46 * (fabs(Ap) + fabs(A) + fabs(r) + fabs(lam)) * inv_u +
                            0x1p-50 * fabs(t);
                        rn = fma(m, u, Fd);                  /* exact: a float */
                        const double ar = fabs(rn);
                        if (fabs(t - m) < 0.5 - tie_eps && ar >= lo + u && ar <= hi - u &&
                            fabs(xd - rn) <= p->eb)
                            fast = 1;
                    }
                }
                if (fast) sy = (uint32_t)(q + p->R);
            }
        }
        if (!fast) {
            ++slow;
            sy = ref_step(xf, r, p, &rn);
            if (sy) {
                K = Kp + ((long long)sy - p->R);
                A = lam + (double)K * p->s;
            } else { /* escape: the lattice restarts at the verbatim value */
                lam = xd;
                K = 0;
                A = lam;
            }
        }
        sym[i] = sy;
        out[i] = (float)rn;
        r = rn;
        Kp = K;
        Ap = A;
    }
    return slow;
}

/* "predicted-q" chain: q is predicted from the lattice index alone (K = rint((x - lam)/s),
 * q = K - Kp), the output is computed with the reference's own arithmetic from that q
 * (cand = RN32(RN64(pred + RN64(q s))): one DADD + the float rounding on the dependent
 * chain), and the prediction is certified off the chain with the reference's quotient
 * (t = RN64(RN64(x - pred) / s) via the reciprocal + the qstep fragility guard): equal
 * rounded quotient => identical step. Failures take the reference step. */
static long chain_plane_q(const float* x, long n, const P* p, uint32_t* sym, float* out) {
    double r = 0.0, lam = 0.0;
    long long Kp = 0;
    long slow = 0;
    for (long i = 0; i < n; ++i) {
        if (g_rebase && i && i % g_rebase == 0) {
            lam = r;
            Kp = 0;
        }
        const float xf = x[i];
        const double xd = xf;
        long long K = (long long)nearbyint((xd - lam) * p->inv_s);
        long long q = K - Kp;
        double rn = 0.0;
        uint32_t sy = 0;
        int fast = 0;
        if (llabs(q) < p->R && fabs(xd) < 0x1p100) {
            const double w = (double)q * p->s;
            const float c = (float)(r + w);
            rn = c;
            /* certification (off the chain): the reference's rounded quotient is q */
            const double d = xd - r;
            const double t = d * p->inv_s;
            const double qd = (double)q;
            const int same = fabs(t - qd) < 0.5 && 0.5 - fabs(t - qd) > fabs(t) * 0x1p-44 + 0x1p-60;
            if (same && isfinite(c) && fabs(xd - rn) <= p->eb) fast = 1;
        }
        if (fast) {
            sy = (uint32_t)(q + p->R);
        } else {
            ++slow;
            sy = ref_step(xf, r, p, &rn);
            if (sy) {
                K = Kp + ((long long)sy - p->R);
            } else {
                lam = xd;
                K = 0;
            }
        }
        sym[i] = sy;
        out[i] = (float)rn;
        r = rn;
        Kp = K;
    }
    return slow;
}

static long ref_plane(const float* x, long n, const P* p, uint32_t* sym, float* out) {
    double r = 0.0;
    for (long i = 0; i < n; ++i) {
        double v;
        sym[i] = ref_step(x[i], r, p, &v);
        out[i] = (float)v;
        r = v;
    }
    return 0;
}

static uint64_t rs = 88172645463325252ull;
static double urand(void) {
    rs ^= rs << 13;
    rs ^= rs >> 7;
    rs ^= rs << 17;
    return ((rs >> 11) + 0.5) * 0x1p-53;
}
static double nrand(void) { return sqrt(-2 * log(urand())) * cos(6.283185307179586 * urand()); }

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 4000000;
    g_rebase = argc > 2 ? atol(argv[2]) : 0;
    g_mode = argc > 3 ? atoi(argv[3]) : 1;
    float* x = malloc(sizeof(float) * n);
    uint32_t *s1 = malloc(4 * n), *s2 = malloc(4 * n);
    float *o1 = malloc(4 * n), *o2 = malloc(4 * n);
    const double ebs[] = {1e-1, 1e-2, 3e-3, 1e-3, 3e-4, 1e-4, 1e-5, 1e-6};
    const char* names[] = {"relu", "dense", "smooth", "lattice", "tiny", "spiky", "huge"};
    long bad_total = 0;
    for (int dist = 0; dist < 7; ++dist) {
        for (int ie = 0; ie < 8; ++ie) {
            const double eb = ebs[ie];
            P p = {eb, 2 * eb, 1.0 / (2 * eb), 32768.0, 32768};
            if (dist == 6) { p.Rd = 1 << 20; p.R = 1 << 20; }
            double sm = 0;
            for (long i = 0; i < n; ++i) {
                double v;
                switch (dist) {
                case 0: v = nrand(); v = v > 0 ? v : 0; break;
                case 1: v = nrand(); break;
                case 2: sm = 0.98 * sm + 0.2 * nrand(); v = sm > 0 ? sm : 0; break;
                case 3: v = floor(nrand() * 50) * p.s + (urand() < 0.5 ? 0.5 * p.s : 0.0); break;
                case 4: v = nrand() * eb * 3; break;
                case 5: v = urand() < 0.01 ? nrand() * 1e4 : nrand(); break;
                default: v = nrand() * 300; break;
                }
                x[i] = (float)v;
            }
            const long plane = 3000;
            long slow = 0, bad = 0;
            for (long a = 0; a < n; a += plane) {
                const long m = n - a < plane ? n - a : plane;
                ref_plane(x + a, m, &p, s1 + a, o1 + a);
                slow += (g_mode ? chain_plane_q : chain_plane)(x + a, m, &p, s2 + a, o2 + a);
            }
            for (long i = 0; i < n; ++i)
                if (s1[i] != s2[i] || memcmp(&o1[i], &o2[i], 4) != 0) {
                    if (bad < 3)
                        printf("  MISMATCH %s eb=%g i=%ld x=%.9g sym %u vs %u out %.9g vs %.9g\n",
                               names[dist], eb, i, x[i], s1[i], s2[i], o1[i], o2[i]);
                    ++bad;
                }
            bad_total += bad;
            printf("%-8s eb=%-6g slow %.5f%%  mismatches %ld\n", names[dist], eb,
                   100.0 * slow / n, bad);
        }
    }
    printf("TOTAL mismatches %ld\n", bad_total);
    return bad_total != 0;
}
