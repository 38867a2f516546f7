// CPU prototype 5: speculative ranges + exact serial walk per plane (design of K2).
//
// phase A (parallel over ranges): range k starts right after an anchor a_k (|x| in the top
//   frequent binade B). Spec chain from the lattice guess g_k = RN32(RN64(lam + K*step)),
//   K = round((x_a - lam)/step), lam = lattice origin (0 at plane start, or the restart value).
//   Per element: spec state s, symbol, robustness margin; collapse bookkeeping.
// phase B (serial per plane, cheap): walk ranges in order with the EXACT offset D = t - s.
//   Only candidate elements are visited (static threshold Tmax); exact steps there.
//   Dense mode when D is too large or too fine. On a lattice disagreement (escape) the rest
//   of the plane is re-speculated from the current exact state (restart) and the walk goes on.
// Verified bit-exact (symbols + exit + sidecar states) against the serial chain.
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
    double pre, q, t;
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
static inline int fexp(double v) {
    int e;
    std::frexp(v, &e);
    return e - 1;
}
static inline int gran(double D) {
    if (D == 0.0) return 100000;
    int e;
    double m = std::frexp(std::fabs(D), &e);
    uint64_t bits = (uint64_t)std::ldexp(m, 53);
    return e - 53 + __builtin_ctzll(bits);
}
static int g_reported = 0;
#define CHECK(tag) do { if (getenv("VERIFY") && !g_reported) { float imp = collapsed ? Tcol : (float)((double)el.s + D); \
   if (imp != tr[i] || ((double)imp - (double)el.s != D && !collapsed)) { g_reported = 1; printf("diverge plane %d i=%ld (%s) kind=%d cand=%d x=%.9g s=%.9g D=%.6g imp=%.9g tr=%.9g sprev=%.9g trprev=%.9g margin=%.3g gran=%d B=%d\n", pl, i, tag, el.kind, el.cand, x[i], el.s, D, imp, tr[i], sprev, i?tr[i-1]:0.f, el.margin, gran(D), B); } } } while (0)
static double gauss() {
    double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0);
    return std::sqrt(-2 * std::log(u)) * std::cos(6.283185307179586 * v);
}

struct Elem {
    float s;
    uint32_t sym;
    double pre;    // spec pre-value (collapse output source)
    float margin;  // robustness margin (decision / acceptance), value units
    int8_t kind;   // 0 normal, 1 collapse, 2 identity in collapsed run, 3 escape
    bool cand;     // static candidate (for |D| <= Tmax)
    double ycol;   // for kind 0 re-expansion / any element after a collapse: last collapse pre
    bool after_col;
    bool tie = false;
    bool nocert = false;
};

struct Cfg {
    int L = 256;
    double Tmax = std::ldexp(1.0, -15);
};

struct PlaneStats {
    long visits = 0, exact = 0, restarts = 0, dense = 0, ranges = 0;
};

// Spec (phase A) for elements [b, e) of the plane from state g (b>0) or plane start (b==0).
static void spec_range(const std::vector<float>& x, long b, long e, float g, int B,
                       std::vector<Elem>& E, const Cfg& cfg) {
    float r = g;
    bool collapsed = false;
    double ycol = 0;
    for (long i = b; i < e; ++i) {
        const double pred = i ? (double)r : 0.0;
        StepOut o = qstep(x[i], pred);
        Elem& el = E[i];
        el.s = o.out;
        el.sym = o.sym;
        el.pre = o.pre;
        el.after_col = collapsed;
        el.ycol = ycol;
        el.cand = false;
        el.tie = false;
        el.nocert = false;
        if (o.sym == 0) {
            el.kind = 3;
            el.margin = 0;
            el.cand = true;
            collapsed = false;
        } else {
            const double dm = (0.5 - std::fabs(o.t - o.q)) * STEP;
            const double am = EB - std::fabs((double)x[i] - (double)o.out);
            el.margin = (float)std::min(dm, am);
            if (el.margin <= 2 * cfg.Tmax) el.cand = true;
            if (std::fabs(o.q) >= (double)RAD - 1) el.cand = true;
            if (o.q == 0 && collapsed) {
                el.kind = 2;
            } else if (std::fabs(o.out) < EB) {
                el.kind = 1;
                collapsed = true;
                ycol = o.pre;
            } else {
                el.kind = 0;
                const int ex = fexp(o.out);
                if (ex > B) el.cand = true;
                {   // exact RN32 tie in the spec pre-value: RNE breaks translation invariance
                    const double half = std::ldexp(1.0, fexp(o.pre) - 24);
                    if (std::fabs(o.pre - (double)o.out) == half) { el.cand = true; el.tie = true; }
                }
                const double a = std::fabs((double)o.out), lo = std::ldexp(1.0, ex);
                if (a - lo <= 2 * cfg.Tmax || 2 * lo - a <= 2 * cfg.Tmax) el.cand = true;
                if (collapsed) {
                    const double dmax = std::ldexp(1.0, fexp(2 * std::max(std::fabs(ycol), 2 * cfg.Tmax)) - 22);
                    const double y = o.pre;
                    const double u = std::ldexp(1.0, fexp(y) - 23);
                    const double fr = std::fabs(std::fmod(std::fabs(y), u) - u / 2);
                    if (!(fr > dmax + std::ldexp(std::fabs(y), -50))) { el.cand = true; el.nocert = true; }
                }
                collapsed = false;
            }
        }
        r = o.out;
    }
}

int main(int argc, char** argv) {
    long P = atol(argv[1]);
    Cfg cfg;
    cfg.L = atoi(argv[2]);
    int mode = atoi(argv[3]);  // 0 dense normal, 1 relu, 2 smooth relu, 3 wide (x100)
    int planes = atoi(argv[4]);
    if (argc > 5) {
        EB = atof(argv[5]);
        STEP = 2 * EB;
    }
    if (argc > 6) cfg.Tmax = atof(argv[6]);
    srand(20201118);
    std::vector<float> x(P), tr(P);
    std::vector<uint32_t> tsym(P);
    std::vector<Elem> E(P);
    PlaneStats st;
    long mism = 0, elems = 0;
    long maxwalk = 0;
    for (int pl = 0; pl < planes; ++pl) {
        for (long i = 0; i < P; ++i) {
            double g = gauss();
            if (mode == 0) x[i] = (float)g;
            else if (mode == 1) x[i] = (float)(g > 0 ? g : 0);
            else if (mode == 3) x[i] = (float)(100 * g);
            else x[i] = 0;
        }
        if (mode == 2) {  // smooth field then relu
            std::vector<double> y(P);
            double acc = 0;
            for (long i = 0; i < P; ++i) { acc = 0.95 * acc + 0.3 * gauss(); y[i] = acc; }
            for (long i = 0; i < P; ++i) x[i] = (float)(y[i] > 0 ? 3 * y[i] : 0);
        }
        {
            float r = 0;
            for (long i = 0; i < P; ++i) {
                StepOut o = qstep(x[i], i ? (double)r : 0.0);
                r = o.out;
                tr[i] = r;
                tsym[i] = o.sym;
            }
        }
        // top frequent binade of the plane (GPU: per tensor from a sample)
        int B = -60;
        for (int e = 20; e >= -60; --e) {
            long c = 0;
            for (long i = 0; i < P; ++i) c += std::fabs(x[i]) >= std::ldexp(1.0, e);
            if (c * 64 >= P) { B = e; break; }
        }
        const double anchor_min = std::ldexp(1.0, B) * (1 + 1.0 / 64);
        std::vector<long> start{0};
        for (long k = 1; k * cfg.L < P; ++k) {
            long a = -1;
            for (long i = k * cfg.L; i < std::min(P, (k + 1) * cfg.L); ++i)
                if (std::fabs(x[i]) >= anchor_min) { a = i; break; }
            if (a >= 0 && a + 1 < P && a + 1 > start.back()) start.push_back(a + 1);
        }
        const long nr = (long)start.size();
        start.push_back(P);
        std::vector<float> guess(nr, 0.0f);
        auto lattice_guess = [&](double lam, long a) {
            const double K = std::round(((double)x[a] - lam) / STEP);
            return (float)(lam + K * STEP);
        };
        std::vector<double> lam(nr, 0.0);
        for (long k = 1; k < nr; ++k) guess[k] = lattice_guess(0.0, start[k] - 1);
        for (long k = 0; k < nr; ++k) spec_range(x, start[k], start[k + 1], guess[k], B, E, cfg);
        // ---- phase B: serial walk ----
        std::vector<uint32_t> sym(P);
        float T = 0;  // exact state before range k (true exit of k-1)
        long walk = 0;
        for (long k = 0; k < nr; ++k) {
            const long b = start[k], e = start[k + 1];
            double D = (double)T - (double)guess[k];
            bool collapsed = false;  // true state is Tcol (spec state collapsed too)
            bool col_wild = false;   // Tcol is not within the certificate bound of s + D
            float Tcol = 0;
            bool restart = false;
            long restart_at = -1;
            for (long i = b; i < e; ++i) {
                const Elem& el = E[i];
                const float sprev = i == b ? guess[k] : E[i - 1].s;
                bool dense = std::fabs(D) > cfg.Tmax || (gran(D) < B - 23);
                if (dense && getenv("WORST") && atoi(getenv("WORST")) == pl) printf("  dense i=%ld k=%ld D=%.4g gran=%d kind=%d s=%.9g\n", i, k, D, gran(D), el.kind, el.s);
                bool visit = el.cand || dense || (i == b) || col_wild;
                if (dense) st.dense++;
                if (!visit) {
                    sym[i] = el.sym;
                    if (el.kind == 1) { collapsed = true; Tcol = (float)(el.pre + D); }
                    else if (el.kind == 0) collapsed = false;
                    CHECK("skip");
                    continue;
                }
                st.visits++;
                walk++;
                if (getenv("WORST") && atoi(getenv("WORST")) == pl) { static long vc[4]; vc[0]+=el.cand; vc[1]+=dense; vc[2]+=col_wild; vc[3]++; if (vc[3] % 5000 == 0) printf("   visits: cand %ld dense %ld wild %ld total %ld (i=%ld k=%ld kind=%d margin=%.3g tie=%d nocert=%d)\n", vc[0],vc[1],vc[2],vc[3], i, k, el.kind, el.margin, el.tie, el.nocert); }
                // true previous state
                const float Tprev = (i == 0) ? 0.0f : (collapsed ? Tcol : (float)((double)sprev + D));
                // can we translate? (full check)
                bool need_exact = true;
                {
                    // dynamic checks
                    double off = collapsed ? std::fabs((double)Tcol - (double)sprev) : std::fabs(D);
                    need_exact = false;
                    if (el.kind == 3) need_exact = true;
                    if (el.margin <= off * (1 + 1e-6) + 1e-30) need_exact = true;
                    if (el.kind == 0) {
                        const int ex = fexp(el.s);
                        if (ex - 23 > gran(D)) need_exact = true;
                        const double a = std::fabs((double)el.s), lo = std::ldexp(1.0, ex);
                        if (a - lo <= std::fabs(D) || 2 * lo - a <= std::fabs(D)) need_exact = true;
                        if (collapsed && (dense || col_wild || el.nocert)) need_exact = true;  // re-expansion w/o certificate
                        if (el.tie) need_exact = true;
                    }
                    if (el.kind == 1 && std::fabs(D) > cfg.Tmax) need_exact = true;
                    if (col_wild) need_exact = true;
                }
                if (!need_exact) {
                    sym[i] = el.sym;
                    if (el.kind == 1) { collapsed = true; Tcol = (float)(el.pre + D); }
                    else if (el.kind == 0) collapsed = false;
                    CHECK("dyn");
                    continue;
                }
                st.exact++;
                StepOut o = qstep(x[i], i == 0 ? 0.0 : (double)Tprev);
                sym[i] = o.sym;
                if (o.sym == 0 || el.kind == 3) {
                    // lattice changes (escape in the true or the spec chain): restart spec
                    // from the exact state after this element
                    collapsed = false;
                    D = (double)o.out - (double)el.s;
                    if (D != 0.0 || (o.sym == 0) != (el.kind == 3)) {
                        restart = true;
                        restart_at = i + 1;
                        T = o.out;
                        break;
                    }
                    // confirmed escape, spec agrees: later ranges move to the lattice of x_i
                    for (long j = k + 1; j < nr; ++j) {
                        if (lam[j] == (double)x[i]) continue;
                        lam[j] = (double)x[i];
                        guess[j] = lattice_guess(lam[j], start[j] - 1);
                        spec_range(x, start[j], start[j + 1], guess[j], B, E, cfg);
                        st.restarts++;
                    }
                } else if ((std::fabs(o.out) < EB) != (el.kind == 1 || el.kind == 2)) {
                    restart = true;
                    restart_at = i + 1;
                    T = o.out;
                    break;
                } else if (std::fabs(o.out) < EB) {
                    collapsed = true;
                    Tcol = o.out;
                    col_wild = std::fabs((double)Tcol - ((double)el.s + D)) > 2 * cfg.Tmax;
                } else {
                    collapsed = false;
                    col_wild = false;
                    D = (double)o.out - (double)el.s;
                }
                CHECK("exact");
            }
            if (restart) {
                st.restarts++;
                // re-speculate the rest of the plane on the lattice of the exact state
                // (GPU: the CTA re-runs phase A for these ranges in parallel)
                long r0 = restart_at;
                // the rest of range k becomes a pseudo-range starting at r0 with exact entry T
                // ranges after k get lattice guesses from lam = T
                start[k] = r0;  // reuse slot k as the remainder (entry exact)
                guess[k] = T;
                if (r0 < e) spec_range(x, r0, e, T, B, E, cfg);
                for (long j = k + 1; j < nr; ++j) {
                    lam[j] = (double)T;
                    guess[j] = lattice_guess((double)T, start[j] - 1);
                    spec_range(x, start[j], start[j + 1], guess[j], B, E, cfg);
                }
                // redo range k from r0 with D = 0 (guess == T)
                --k;
                // next iteration computes D = T - guess[k] = 0
                continue;
            }
            const long last = e - 1;
            T = collapsed ? Tcol : (float)((double)E[last].s + D);
        }
        if (getenv("WORST") && walk > P / 3) printf("plane %d walk %ld B=%d nr=%ld\n", pl, walk, B, nr);
        maxwalk = std::max(maxwalk, walk);
        st.ranges += nr;
        elems += P;
        { long m0 = mism; for (long i = 0; i < P; ++i) mism += sym[i] != tsym[i];
          if (mism != m0 && getenv("SHOW")) { for (long i = 0; i < P; ++i) if (sym[i] != tsym[i]) {
              printf("plane %d first mismatch at %d x=%.9g kind=%d cand=%d spec=%u true=%u got=%u s=%.9g tr=%.9g prev s=%.9g tr=%.9g\n", pl, (int)i, x[i], E[i].kind, E[i].cand, E[i].sym, tsym[i], sym[i], E[i].s, tr[i], i?E[i-1].s:0, i?tr[i-1]:0); break; } } }
        if (T != tr[P - 1]) mism++;
    }
    printf("P=%ld L=%d mode=%d eb=%g: MISMATCH %ld | visits/elem %.4f exact/elem %.4f dense/elem %.4f restarts/plane %.3f | max walk %ld (%.2f/elem)\n",
           P, cfg.L, mode, EB, mism, (double)st.visits / elems, (double)st.exact / elems,
           (double)st.dense / elems, (double)st.restarts / planes, maxwalk, (double)maxwalk / P);
}
