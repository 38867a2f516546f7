// CPU prototype 4 (design validation for the K2 quantiser): "speculate -> scan -> certify ->
// repair" for the exact PrevValue chain of the reference (src/codec.cpp:76-104).
//
//  phase A  : ranges start right after an anchor (element in the top frequent binade B); the
//             speculative chain starts from the ideal lattice value of the anchor. Per element
//             we keep the spec state, the symbol, and per-element robustness margins.
//  scan     : predicted true offset D_k of range k = prefix sum of (spec anchor output of
//             range k-1 - guess of range k) (+ corrections from the previous round).
//  walk     : per range, given D_k: visit candidate events only (fragile decision /
//             acceptance margins, binade edges, coarse elements, escapes, collapse pairs
//             without certificate); exact step there; D := t - s afterwards.
//  iterate  : if a walk changes D, the correction is prefix-summed into later ranges; repeat.
// Checks bit-exactness of every symbol and of the exit against the serial chain.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static double EB = 1e-3, STEP = 2e-3;
static int64_t RAD = 32768;

struct StepOut {
    uint32_t sym;
    float out;
    double pre;  // RN64(pred + q*step) (NaN for escape)
    double q;
    double t;    // (x - pred)/step
};

static inline StepOut qstep(float xf, double pred) {
    StepOut o;
    const double orig = xf;
    o.t = (orig - pred) / STEP;
    o.q = std::round(o.t);
    o.pre = NAN;
    if (std::fabs(o.q) < (double)RAD) {
        const double y = pred + o.q * STEP;
        const float cand = (float)y;
        if (std::isfinite(cand) && std::fabs(orig - (double)cand) <= EB) {
            o.sym = (uint32_t)((int64_t)o.q + RAD);
            o.out = cand;
            o.pre = y;
            return o;
        }
    }
    o.sym = 0;
    o.out = xf;
    return o;
}

static inline int fexp(float v) {  // binade exponent of a nonzero finite float
    int e;
    std::frexp(v, &e);
    return e - 1;
}

// exponent of the lowest set bit of D (granularity); large when D == 0
static inline int gran(double D) {
    if (D == 0.0) return 10000;
    int e;
    double m = std::frexp(std::fabs(D), &e);  // D = m * 2^e, m in [0.5,1)
    uint64_t bits = (uint64_t)std::ldexp(m, 53);
    return e - 53 + __builtin_ctzll(bits);
}

static double gauss() {
    double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0);
    return std::sqrt(-2 * std::log(u)) * std::cos(6.283185307179586 * v);
}

long why[8];
struct Stats {
    long ranges = 0, cand = 0, exact = 0, rounds = 0, maxrounds = 0, elems = 0, cand_lim = 0;
};

// Per-element phase-A data.
struct Elem {
    float s;        // spec state after element
    uint32_t sym;
    float x;
    double pre;     // spec pre-value
    float margin;   // min(decision margin, acceptance margin) in value units
    int8_t kind;    // 0 normal, 1 collapse (tiny output), 2 zero-identity, 3 escape
    bool cert;      // re-expansion certificate (for kind 0 after a collapse)
};

int main(int argc, char** argv) {
    long P = atol(argv[1]);
    int L = atoi(argv[2]);
    int relu = atoi(argv[3]);
    int planes = atoi(argv[4]);
    if (argc > 5) {
        EB = atof(argv[5]);
        STEP = 2 * EB;
    }
    double Tmax = argc > 6 ? atof(argv[6]) : std::ldexp(1.0, -15);
    srand(99);
    std::vector<float> x(P), tr(P);
    std::vector<uint32_t> tsym(P);
    Stats st;
    long mism = 0;
    for (int pl = 0; pl < planes; ++pl) {
        for (long i = 0; i < P; ++i) {
            double g = gauss();
            x[i] = (float)(relu ? (g > 0 ? g : 0) : g);
        }
        // serial truth
        {
            float r = 0;
            for (long i = 0; i < P; ++i) {
                StepOut o = qstep(x[i], i ? (double)r : 0.0);
                r = o.out;
                tr[i] = r;
                tsym[i] = o.sym;
            }
        }
        // top frequent binade B: largest e with count(|x| >= 2^e) >= P/64
        int B = -30;
        for (int e = 10; e >= -30; --e) {
            long c = 0;
            for (long i = 0; i < P; ++i) c += std::fabs(x[i]) >= std::ldexp(1.0, e);
            if (c * 64 >= P) {
                B = e;
                break;
            }
        }
        const double anchor_min = std::ldexp(1.0, B) * (1 + 1.0 / 64);
        // ranges: range 0 starts at 0; range k>0 starts after the first anchor >= k*L
        std::vector<long> start{0};
        for (long k = 1; k * L < P; ++k) {
            long a = -1;
            for (long i = k * L; i < std::min(P, (k + 1) * L); ++i)
                if (std::fabs(x[i]) >= anchor_min) {
                    a = i;
                    break;
                }
            if (a >= 0 && a + 1 < P && a + 1 > start.back()) start.push_back(a + 1);
        }
        const long nr = (long)start.size();
        start.push_back(P);
        std::vector<Elem> E(P);
        std::vector<float> guess(nr);
        // ---- phase A ----
        for (long k = 0; k < nr; ++k) {
            float r = 0;
            if (k > 0) r = (float)(std::round((double)x[start[k] - 1] / STEP) * STEP);
            guess[k] = r;
            bool collapsed = false;
            double ycol = 0;
            for (long i = start[k]; i < start[k + 1]; ++i) {
                const double pred = i ? (double)r : 0.0;
                StepOut o = qstep(x[i], pred);
                Elem& e = E[i];
                e.x = x[i];
                e.s = o.out;
                e.sym = o.sym;
                e.pre = o.pre;
                e.cert = true;
                if (o.sym == 0) {
                    e.kind = 3;
                    e.margin = 0;
                    collapsed = false;
                } else {
                    const double dm = (0.5 - std::fabs(o.t - o.q)) * STEP;
                    const double am = EB - std::fabs((double)x[i] - (double)o.out);
                    e.margin = (float)std::min(dm, am);
                    if (o.q == 0 && collapsed) {
                        e.kind = 2;  // identity inside a zero run
                    } else if (std::fabs(o.out) < EB) {
                        e.kind = 1;  // collapse
                        collapsed = true;
                        ycol = o.pre;
                    } else {
                        e.kind = 0;
                        if (collapsed) {
                            // re-expansion certificate for any |D| <= Tmax
                            const double dmax = std::ldexp(1.0, fexp((float)(2 * std::max(std::fabs(ycol), Tmax))) - 22);
                            const double y = o.pre;
                            const int ey = fexp((float)y);
                            const double u = std::ldexp(1.0, ey - 23);
                            const double fr = std::fabs(std::fmod(std::fabs(y), u) - u / 2);
                            e.cert = fr > dmax + std::ldexp(std::fabs(y), -50);
                        }
                        collapsed = false;
                    }
                }
                r = o.out;
            }
        }
        // ---- scan + walk rounds ----
        std::vector<double> Din(nr, 0.0), Dout(nr, 0.0), corr(nr, 0.0);
        std::vector<uint32_t> sym(P);
        std::vector<float> exitv(nr);
        int rounds = 0;
        for (;;) {
            ++rounds;
            // scan: predicted offsets
            if (rounds == 1) {
                for (long k = 1; k < nr; ++k)
                    Din[k] = Din[k - 1] + ((double)E[start[k] - 1].s - (double)guess[k]);
            } else {
                // defect = predecessor's walked exit - entry used; prefix-summed (translation)
                double acc = 0;
                for (long k = 1; k < nr; ++k) {
                    acc += (double)exitv[k - 1] - ((double)guess[k] + Din[k]);
                    Din[k] += acc;
                }
            }
            bool changed = false;
            if (getenv("DBG") && pl == atoi(getenv("DBG"))) {
                for (long k = 1; k < nr && k < 40; ++k) {
                    double tD = (double)tr[start[k] - 1] - (double)guess[k];
                    printf("round %d k=%ld start=%ld x[a]=%g guess=%.9g Din=%.3g trueD=%.3g %s\n", rounds, k, start[k], x[start[k]-1], guess[k], Din[k], tD, Din[k]==tD?"":"  <--");
                }
            }
            for (long k = 0; k < nr; ++k) {
                double D = Din[k];
                // true state before range = guess + D (range 0: exact 0)
                float T = k == 0 ? 0.0f : (float)((double)guess[k] + D);
                bool collapsed = false;  // true state currently RN32(ycol + Dc)
                float Tcol = 0;
                for (long i = start[k]; i < start[k + 1]; ++i) {
                    const Elem& e = E[i];
                    const float sprev = i == start[k] ? guess[k] : E[i - 1].s;
                    const float Tprev = (i == 0) ? 0.0f : (collapsed ? Tcol : (float)((double)sprev + D));
                    bool cand = std::fabs(D) > Tmax;  // beyond certified range: check everything
                    if (cand) why[0]++;
                    if (e.kind == 3) { cand = true; why[1]++; }
                    if (e.kind == 0 || e.kind == 1 || e.kind == 2) {
                        double off = std::fabs(D);
                        if (collapsed) off = std::fabs((double)Tcol - (double)sprev);
                        if (e.margin <= off * (1 + 1e-6) + 1e-30) { cand = true; why[2]++; }
                    }
                    if (e.kind == 0) {
                        const int ex = fexp(e.s);
                        if (ex - 23 > gran(D)) { cand = true; why[3]++; }  // coarser than D's granularity
                        const double lo = std::ldexp(1.0, ex), hi = 2 * lo;
                        const double a = std::fabs((double)e.s);
                        if (a - lo <= std::fabs(D) || hi - a <= std::fabs(D)) { cand = true; why[4]++; }
                        if (!e.cert) { cand = true; why[5]++; }
                    }
                    if (i == start[k] && k > 0) {
                        // D must be a multiple of the anchor grid; else treat as event
                        double u = std::ldexp(1.0, B - 23);
                        if (std::fmod(std::fabs(D), u) != 0.0) { cand = true; why[6]++; }
                    }
                    if (cand) st.cand++;
                    bool dbg = getenv("DBG") && pl == atoi(getenv("DBG")) && getenv("RNG") && k == atoi(getenv("RNG")) && rounds == 1;
                    if (cand) {
                        st.exact++;
                        StepOut o = qstep(e.x, i == 0 ? 0.0 : (i == start[0] ? 0.0 : (double)Tprev));
                        if (i == 0) o = qstep(e.x, 0.0);
                        sym[i] = o.sym;
                        if (o.sym == 0) {
                            collapsed = false;
                            D = (double)o.out - (double)e.s;
                        } else if (e.kind == 1 || e.kind == 2) {
                            collapsed = true;
                            Tcol = o.out;
                            D = D;  // keep coarse offset
                        } else {
                            collapsed = false;
                            D = (double)o.out - (double)e.s;
                        }
                    } else {
                        sym[i] = e.sym;
                        if (e.kind == 1) {
                            collapsed = true;
                            Tcol = (float)(e.pre + D);
                        } else if (e.kind == 2) {
                            // identity
                        } else {
                            collapsed = false;
                        }
                    }
                    if (dbg) { float implied = collapsed ? Tcol : (float)((double)e.s + D); printf("  i=%ld x=%.9g kind=%d s=%.9g D=%.3g implied=%.9g true=%.9g cand=%d margin=%.3g %s\n", i, e.x, e.kind, e.s, D, implied, tr[i], cand, e.margin, implied==tr[i]?"":"<--"); }
                }
                if (getenv("DBG") && pl == atoi(getenv("DBG")) && getenv("RNG") && k == atoi(getenv("RNG")) && rounds == 1) {}
                const long last = start[k + 1] - 1;
                float ex = collapsed ? Tcol : (float)((double)E[last].s + D);
                if (rounds > 1 && ex != exitv[k]) changed = true;
                if (rounds == 1) changed = true;
                exitv[k] = ex;
                Dout[k] = D;
            }
            if (!changed) break;
            if (rounds > 50) break;
        }
        st.rounds += rounds;
        st.maxrounds = std::max<long>(st.maxrounds, rounds);
        st.ranges += nr;
        st.elems += P;
        { long m0 = mism; for (long i = 0; i < P; ++i) mism += sym[i] != tsym[i];
          if (mism != m0 && getenv("SHOW")) { printf("plane %d mism %ld rounds %d\n", pl, mism - m0, rounds);
            for (long i = 0; i < P; ++i) if (sym[i] != tsym[i]) { long k=0; while (start[k+1] <= i) ++k; printf("  first at %ld (range %ld start %ld) x=%g kind=%d spec=%u true=%u got=%u\n", i, k, start[k], x[i], E[i].kind, E[i].sym, tsym[i], sym[i]); break; } } }
        if (exitv[nr - 1] != tr[P - 1]) mism++;
    }
    printf("why: |D|>T %ld esc %ld margin %ld coarse %ld binade %ld cert %ld grid %ld\n", why[0],why[1],why[2],why[3],why[4],why[5],why[6]);
    printf("P=%ld L=%d relu=%d eb=%g Tmax=%g: mismatches %ld | rounds mean %.2f max %ld | candidates/elem %.4f exact/elem %.4f | elems/range %.1f\n",
           P, L, relu, EB, Tmax, mism, (double)st.rounds / planes, st.maxrounds, (double)st.cand / st.elems / ((double)st.rounds / planes),
           (double)st.exact / st.elems / ((double)st.rounds / planes), (double)st.elems / st.ranges);
}
