// Host engine + C ABI (include/dreg_cuda.h) for the B200 registration path.
//
// Owns device workspaces (one per grid size, reused across calls), builds the
// per-axis FFT plans and their device tables, issues the registration launch
// sequence -- captured once into a CUDA graph per (workspace, config) and replayed
// -- and converts between the reference's AoS host layout and the device SoA one.
// No compute happens on the host: every numerical step is an sm_100a kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "dreg_cuda.h"
#include "launch.h"

using namespace dregb;

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

struct Status {
    int code = DREG_OK;
    std::string msg;
};

#define CK(expr)                                                                     \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess)                                                       \
            throw CudaFail(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
    } while (0)

struct CudaFail {
    std::string msg;
    explicit CudaFail(std::string m) : msg(std::move(m)) {}
};
struct ArgFail {
    std::string msg;
    explicit ArgFail(std::string m) : msg(std::move(m)) {}
};
struct NumFail {
    std::string msg;
    explicit NumFail(std::string m) : msg(std::move(m)) {}
};

// Guard-band mode (DREG_GUARD=1; compute-sanitizer is unavailable on the GPU pool):
// every device buffer gets kGuard bytes of a fixed pattern on both sides, and
// dreg_cuda_check_guards() / the end of every registration verify them -- any kernel
// write past either end of any workspace buffer is reported (tests/test_guard.py).
constexpr size_t kGuard = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;
inline bool guard_mode() {
    static const int g = [] {
        const char* v = std::getenv("DREG_GUARD");
        return v && *v ? std::atoi(v) : 0;
    }();
    return g != 0;
}

template <class T>
struct DevArray {
    T* p = nullptr;
    size_t n = 0;
    unsigned char* base = nullptr;  // allocation start (guard mode: p - kGuard)
    DevArray() = default;
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    ~DevArray() { release(); }
    void release() {
        if (base) cudaFree(base);
        base = nullptr;
        p = nullptr;
    }
    void alloc(size_t count) {
        release();
        n = count;
        if (!count) return;
        const size_t bytes = sizeof(T) * count;
        if (guard_mode()) {
            CK(cudaMalloc(&base, bytes + 2 * kGuard));
            CK(cudaMemset(base, kGuardByte, kGuard));
            CK(cudaMemset(base + kGuard + bytes, kGuardByte, kGuard));
            p = reinterpret_cast<T*>(base + kGuard);
        } else {
            CK(cudaMalloc(&base, bytes));
            p = reinterpret_cast<T*>(base);
        }
    }
    // true when both guard bands still hold the pattern (always true outside guard mode)
    bool guards_intact() const {
        if (!guard_mode() || !base) return true;
        std::vector<unsigned char> h(kGuard);
        for (const unsigned char* g : {base, base + kGuard + sizeof(T) * n}) {
            CK(cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost));
            for (unsigned char b : h)
                if (b != kGuardByte) return false;
        }
        return true;
    }
};

// ---- line FFT plan (host) ------------------------------------------------------
AxisPlan make_plan(int n) {
    AxisPlan P{};
    P.n = n;
    int rem = n, s = 0;
    while (rem > 1) {
        int r;
        if (rem % 8 == 0) r = 8;
        else if (rem % 4 == 0) r = 4;
        else if (rem % 2 == 0) r = 2;
        else if (rem % 3 == 0) r = 3;
        else if (rem % 5 == 0) r = 5;
        else if (rem % 7 == 0) r = 7;
        else {
            r = 11;
            while (rem % r) r += 2;
        }
        if (r > kMaxRadix) throw ArgFail("FFT length " + std::to_string(n) + " has a prime factor > 64");
        if (s >= kMaxStages) throw ArgFail("FFT length " + std::to_string(n) + " needs too many stages");
        P.radix[s++] = r;
        rem /= r;
    }
    P.nst = s;
    int ns = n;
    for (int i = 0; i < s; ++i) {
        P.n1[i] = ns / P.radix[i];
        P.tws[i] = n / ns;
        P.fn1[i].init((unsigned)P.n1[i]);
        ns = P.n1[i];
    }
    return P;
}

// frequency held at position `pos` after the DIF stages (digit reversal)
int freq_of_pos(const AxisPlan& P, int pos) {
    int f = 0, mult = 1, p = pos;
    for (int s = 0; s < P.nst; ++s) {
        const int k2 = p / P.n1[s];
        p -= k2 * P.n1[s];
        f += mult * k2;
        mult *= P.radix[s];
    }
    return f;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

float2 w_of(long num, long den) {  // exp(-2 pi i num/den), computed in double
    long q = num % den;
    if (q < 0) q += den;
    const double a = -2.0 * kPi * (double)q / (double)den;
    return make_float2((float)std::cos(a), (float)std::sin(a));
}

float one_minus_cos(int k, int n) {  // 1 - cos(2 pi k / n) = 2 sin^2(pi k / n); exactly 0 at k = 0
    if (k == 0) return 0.f;
    const double s = std::sin(kPi * (double)k / (double)n);
    return (float)(2.0 * s * s);
}

// ---- geometry + device tables for one grid -------------------------------------
struct Geometry {
    int M = 0, Ny = 0, Nz = 0, hx = 0;
    long long N = 0, lines = 0;
    int L = 0, odd = 0, TL = 0, TLp = 0, PM = 0, PY = 0, xvec = 1;
    AxisPlan px{}, py{}, pz{};
    DevArray<float2> twx, xtw, twy, twz;
    DevArray<int> xpos;
    DevArray<float> sx, sy, sz, sy_fast, sz_fast;
    DevArray<double2> twx64, xtw64, twy64, twz64;  // precise-mode tables
    DevArray<double> sx64, sy64, sz64;
    DevArray<double> cx64, cy64, cz64;  // reference axis cosines for the precise multiplier
    DevArray<double> cy64_fast, cz64_fast;  // ... at the cluster plane kernel's positions
    int fast = 0, prefetch = 1;
    size_t xsmem = 0, psmem = 0;

    void build(dreg_dims3 d) {
        M = d.x;
        Ny = d.y;
        Nz = d.z;
        hx = M / 2 + 1;
        N = (long long)M * Ny * Nz;
        lines = (long long)Ny * Nz;
        odd = (M % 2 != 0) || M < 2;
        L = odd ? M : M / 2;
        px = make_plan(L);
        py = make_plan(Ny);
        pz = make_plan(Nz);
        PM = (L % 2 == 0) ? L + 1 : L;
        PY = (Ny % 2 == 0) ? Ny + 1 : Ny;
        TL = env_int("DREG_TL", 32);
        xvec = env_int("DREG_XVEC", 2);
        {
            int t = 4;  // power of two (the x-pass index math uses shifts)
            while (t * 2 <= std::max(TL, 4) && t < 64) t *= 2;
            TL = t;
        }
        while (TL > 4 && xpass_smem_bytes(L, hx, TL, PM) > 110 * 1024) TL /= 2;
        xsmem = xpass_smem_bytes(L, hx, TL, PM);
        TLp = TL;  // precise (double2) generic x-pass: same budget, half the lines
        while (TLp > 4 && xpass_smem_bytes_c(L, hx, TLp, PM, sizeof(double2)) > 110 * 1024) TLp /= 2;
        if ((lines + TLp - 1) / TLp > kMaxPartials) TLp = TL;  // keep the partial-sum slots in range
        psmem = plane_smem_bytes(Ny, Nz, PY);
        if (xsmem > 227 * 1024) throw ArgFail("x extent too large for the shared-memory x-pass");
        if ((lines + TL - 1) / TL > kMaxPartials) throw ArgFail("grid has too many x-lines");

        std::vector<float2> h(L);
        for (int e = 0; e < L; ++e) h[e] = w_of(e, L);
        up(twx, h);
        std::vector<float2> hxw(hx + 1);
        for (int k = 0; k <= hx; ++k) hxw[k] = w_of(k, M);
        up(xtw, hxw);
        std::vector<int> hp(L);
        for (int pos = 0; pos < L; ++pos) hp[freq_of_pos(px, pos)] = pos;
        up(xpos, hp);
        h.assign(Ny, {});
        for (int e = 0; e < Ny; ++e) h[e] = w_of(e, Ny);
        up(twy, h);
        h.assign(Nz, {});
        for (int e = 0; e < Nz; ++e) h[e] = w_of(e, Nz);
        up(twz, h);
        std::vector<float> s(hx);
        for (int p = 0; p < hx; ++p) s[p] = one_minus_cos(p, M);
        up(sx, s);
        s.assign(Ny, 0.f);
        for (int pos = 0; pos < Ny; ++pos) s[pos] = one_minus_cos(freq_of_pos(py, pos), Ny);
        up(sy, s);
        s.assign(Nz, 0.f);
        for (int pos = 0; pos < Nz; ++pos) s[pos] = one_minus_cos(freq_of_pos(pz, pos), Nz);
        up(sz, s);
        {  // fp64 copies of the twiddles / symbol tables for the precise mode
            auto w64 = [](long num, long den) {
                long q = num % den;
                if (q < 0) q += den;
                const double a = -2.0 * kPi * (double)q / (double)den;
                return make_double2(std::cos(a), std::sin(a));
            };
            auto s64 = [](int k, int n) {
                if (k == 0) return 0.0;
                const double t = std::sin(kPi * (double)k / (double)n);
                return 2.0 * t * t;
            };
            std::vector<double2> hd(L);
            for (int e = 0; e < L; ++e) hd[e] = w64(e, L);
            up(twx64, hd);
            hd.assign(hx + 1, {});
            for (int k = 0; k <= hx; ++k) hd[k] = w64(k, M);
            up(xtw64, hd);
            hd.assign(Ny, {});
            for (int e = 0; e < Ny; ++e) hd[e] = w64(e, Ny);
            up(twy64, hd);
            hd.assign(Nz, {});
            for (int e = 0; e < Nz; ++e) hd[e] = w64(e, Nz);
            up(twz64, hd);
            std::vector<double> sd(hx);
            for (int p = 0; p < hx; ++p) sd[p] = s64(p, M);
            up(sx64, sd);
            sd.assign(Ny, 0.0);
            for (int pos = 0; pos < Ny; ++pos) sd[pos] = s64(freq_of_pos(py, pos), Ny);
            up(sy64, sd);
            sd.assign(Nz, 0.0);
            for (int pos = 0; pos < Nz; ++pos) sd[pos] = s64(freq_of_pos(pz, pos), Nz);
            up(sz64, sd);
            // axis_cosines (regularizer.cpp:24-31): the same expression, c[0] forced to 1
            auto cos_ref = [](int k, int n) { return k == 0 ? 1.0 : std::cos(2.0 * kPi * k / n); };
            sd.assign(hx, 0.0);
            for (int p = 0; p < hx; ++p) sd[p] = cos_ref(p, M);
            up(cx64, sd);
            sd.assign(Ny, 0.0);
            for (int pos = 0; pos < Ny; ++pos) sd[pos] = cos_ref(freq_of_pos(py, pos), Ny);
            up(cy64, sd);
            sd.assign(Nz, 0.0);
            for (int pos = 0; pos < Nz; ++pos) sd[pos] = cos_ref(freq_of_pos(pz, pos), Nz);
            up(cz64, sd);
            if (plane_cluster_fast64_supported(Ny, Nz)) {  // splits y: 16 x Ny/16, z: Nz/16 x 16
                auto split2 = [](int n, int r1) {
                    AxisPlan q{};
                    q.n = n;
                    q.nst = 2;
                    q.radix[0] = r1;
                    q.radix[1] = n / r1;
                    q.n1[0] = q.radix[1];
                    q.n1[1] = 1;
                    return q;
                };
                const AxisPlan fy = split2(Ny, 16), fz = split2(Nz, Nz / 16);
                sd.assign(Ny, 0.0);
                for (int pos = 0; pos < Ny; ++pos) sd[pos] = cos_ref(freq_of_pos(fy, pos), Ny);
                up(cy64_fast, sd);
                sd.assign(Nz, 0.0);
                for (int pos = 0; pos < Nz; ++pos) sd[pos] = cos_ref(freq_of_pos(fz, pos), Nz);
                up(cz64_fast, sd);
            }
        }
        // 1 = plane_fast_kernel; >= 2 (default 3) = register-blocked plane_reg_kernel where
        // it applies (first stages radix 8 on y and Nz / 16 on z, second stages in smem)
        fast = plane_fast_supported(Ny, Nz) ? env_int("DREG_FAST_PLANE", 3) : 0;
        if (fast >= 2 && !plane_reg_supported(Ny, Nz)) fast = 1;
        prefetch = env_int("DREG_PREFETCH", 0);
        if (!fast && plane_cluster_fast_supported(Ny, Nz)) {
            // position tables of the cluster plane kernel's splits (y: 16 x Ny/16, z: Nz/16 x 16)
            auto split2 = [](int n, int r1) {
                AxisPlan q{};
                q.n = n;
                q.nst = 2;
                q.radix[0] = r1;
                q.radix[1] = n / r1;
                q.n1[0] = q.radix[1];
                q.n1[1] = 1;
                return q;
            };
            const AxisPlan fy = split2(Ny, 16), fz = split2(Nz, Nz / 16);
            s.assign(Ny, 0.f);
            for (int pos = 0; pos < Ny; ++pos) s[pos] = one_minus_cos(freq_of_pos(fy, pos), Ny);
            up(sy_fast, s);
            s.assign(Nz, 0.f);
            for (int pos = 0; pos < Nz; ++pos) s[pos] = one_minus_cos(freq_of_pos(fz, pos), Nz);
            up(sz_fast, s);
        }
        if (fast) {
            // tables for the two-stage split R1 x R2 of the specialised kernel
            auto split = [](int n, int r1) {
                AxisPlan q{};
                q.n = n;
                q.nst = 2;
                q.radix[0] = r1;
                q.radix[1] = n / q.radix[0];
                q.n1[0] = q.radix[1];
                q.n1[1] = 1;
                return q;
            };
            const AxisPlan fy = split(Ny, plane_fast_r1(Ny)), fz = split(Nz, fast >= 2 ? Nz / 16 : plane_fast_r1(Nz));
            s.assign(Ny, 0.f);
            for (int pos = 0; pos < Ny; ++pos) s[pos] = one_minus_cos(freq_of_pos(fy, pos), Ny);
            up(sy_fast, s);
            s.assign(Nz, 0.f);
            for (int pos = 0; pos < Nz; ++pos) s[pos] = one_minus_cos(freq_of_pos(fz, pos), Nz);
            up(sz_fast, s);
        }
    }

    template <class T>
    static void up(DevArray<T>& d, const std::vector<T>& h) {
        d.alloc(h.size());
        CK(cudaMemcpy(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    }
};

// ---- workspace: all per-chunk device state --------------------------------------
struct Workspace {
    Geometry geo;
    int P = 0;       // pair capacity
    int diag_iters = 0;
    DevArray<float> V, BH, WP, BP, G, D, I0, I1, PHI0, PHI1, W0, W1;
    DevArray<float2> S;
    DevArray<float2> S2;  // scratch spectrum for the logged objective (solve_velocity only; lazy)
    DevArray<double2> S64, S264;  // fp64 spectrum (+ scratch) of the precise mode (lazy)
    DevArray<PairState> st;
    DevArray<double> part, diag, energy;
    DevArray<float> stage_t, stage_s, stage3, phi_soa, warped;
    DevArray<const float*> tgt_tab, src_tab;
    DevArray<float*> phi_tab, warped_tab;
    DevArray<unsigned int> counter;
    DevArray<double> scal;   // small scalar outputs
    DevArray<float> fscal;
    std::map<std::string, std::pair<cudaGraphExec_t, int>> graphs;

    ~Workspace() { clear_graphs(); }
    void clear_graphs() {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
        graphs.clear();
    }

    // device bytes per pair: the ADMM state V BH WP BP G (15 words) + D, I0, I1, PHI x2,
    // WARPED x2 (11) + the x-spectrum; host-buffer batches add the double-buffered staging
    // (stage_t, stage_s, stage3, warped x2 and phi_soa: 15 words), allocated lazily
    static size_t bytes_per_pair(const Geometry& g, bool host) {
        return sizeof(float) * (size_t)g.N * (26 + (host ? 15 : 0)) + sizeof(float2) * 3 * (size_t)g.hx * g.lines +
               sizeof(double) * 3 * kMaxPartials;
    }

    void ensure_staging() {  // host-path staging (register_batch from host buffers, AoS I/O)
        if (stage3.p) return;
        const size_t N = (size_t)geo.N;
        stage_t.alloc(2 * P * N);
        stage_s.alloc(2 * P * N);
        stage3.alloc(2 * P * 3 * N);
        phi_soa.alloc(P * 3 * N);
        warped.alloc(2 * P * N);
    }

    // guard-band check of every buffer (DREG_GUARD); returns the first corrupted name
    const char* corrupted_buffer() const {
#define DREG_G(b) \
    if (!b.guards_intact()) return #b;
        DREG_G(V) DREG_G(BH) DREG_G(WP) DREG_G(BP) DREG_G(G) DREG_G(D) DREG_G(I0) DREG_G(I1) DREG_G(PHI0)
        DREG_G(PHI1) DREG_G(W0) DREG_G(W1) DREG_G(S) DREG_G(S2) DREG_G(S64) DREG_G(S264) DREG_G(st) DREG_G(part)
        DREG_G(diag) DREG_G(energy) DREG_G(stage_t) DREG_G(stage_s) DREG_G(stage3) DREG_G(phi_soa) DREG_G(warped)
        DREG_G(tgt_tab) DREG_G(src_tab) DREG_G(phi_tab) DREG_G(warped_tab) DREG_G(counter) DREG_G(scal) DREG_G(fscal)
#undef DREG_G
        return nullptr;
    }

    void alloc(dreg_dims3 d, int pairs) {
        static unsigned long long next_id = 1;
        id = next_id++;
        geo.build(d);
        P = pairs;
        const size_t N = (size_t)geo.N;
        V.alloc(P * 3 * N);
        // the two dual-iterate buffers double as the spectral-state iteration's U_j / U_{j-1}
        // ([3][hx][lines] complex = 3 (M + 2) lines floats per pair)
        const size_t bwords = (size_t)P * 3 * (size_t)(geo.M + 2) * (size_t)geo.lines;
        BH.alloc(std::max((size_t)P * 3 * N, bwords));
        WP.alloc(P * 3 * N);
        BP.alloc(std::max((size_t)P * 3 * N, bwords));
        G.alloc(P * 3 * N);
        D.alloc(P * N);
        I0.alloc(P * N);
        I1.alloc(P * N);
        PHI0.alloc(P * 3 * N);
        PHI1.alloc(P * 3 * N);
        W0.alloc(P * N);
        W1.alloc(P * N);
        S.alloc((size_t)P * 3 * geo.hx * geo.lines);
        st.alloc(P);
        part.alloc((size_t)P * 3 * kMaxPartials);
        energy.alloc(P);
        tgt_tab.alloc(P);
        src_tab.alloc(P);
        phi_tab.alloc(P);
        warped_tab.alloc(P);
        counter.alloc(4);
        CK(cudaMemset(counter.p, 0, sizeof(unsigned int) * 4));
        CK(cudaMemset(st.p, 0, sizeof(PairState) * P));
        scal.alloc(8);
        fscal.alloc(2 + 2 * kMaxPartials);
        clear_graphs();
    }

    void ensure_s64() {  // precise mode's fp64 spectrum (allocated before any graph capture)
        if (!S64.p) S64.alloc(S.n);
    }

    void ensure_diag(int iters) {
        if (iters > diag_iters) {
            diag.alloc((size_t)P * iters * 3);
            diag_iters = iters;
            clear_graphs();
        }
    }

    PairState* st_shared = nullptr;  // set on coarser pyramid levels: state lives in the finest workspace
    unsigned long long id = 0;       // allocation generation (graph cache key)

    Fields fields(bool with_diag) const {
        Fields F{};
        F.M = geo.M;
        F.Ny = geo.Ny;
        F.Nz = geo.Nz;
        F.hx = geo.hx;
        F.N = geo.N;
        F.lines = geo.lines;
        F.V = V.p;
        F.BH = BH.p;
        F.WP = WP.p;
        F.BP = BP.p;
        F.G = G.p;
        F.D = D.p;
        F.T = I0.p;
        F.S = S.p;
        F.S64 = S64.p;
        F.st = st_shared ? st_shared : st.p;
        F.part = part.p;
        F.diag = with_diag ? diag.p : nullptr;
        F.diag_stride = diag_iters;
        return F;
    }

    RegBuffers regbufs() const {
        RegBuffers R{};
        R.I0 = I0.p;
        R.I1 = I1.p;
        R.PHI[0] = PHI0.p;
        R.PHI[1] = PHI1.p;
        R.WARPED[0] = W0.p;
        R.WARPED[1] = W1.p;
        R.tgt_in = tgt_tab.p;
        R.src_in = src_tab.p;
        R.phi_out = phi_tab.p;
        R.warped_out = warped_tab.p;
        R.tmpA = D.p;   // prep scratch aliases D / G (free before the first solve)
        R.tmpB = G.p;
        return R;
    }

    VolGeom vg() const { return VolGeom{geo.M, geo.Ny, geo.Nz, geo.N}; }
};

bool same_dims(const Geometry& g, dreg_dims3 d) { return g.M == d.x && g.Ny == d.y && g.Nz == d.z; }

}  // namespace

struct dreg_cuda_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    int chunk = 0;
    int use_graphs = 1;
    int precision = 0;  // 0 auto (fp64 spectral arithmetic for solves > 100 iterations), 1 fp32, 2 fp64
    std::map<std::tuple<int, int, int>, std::unique_ptr<Workspace>> wss;  // one per grid size
    Workspace* last = nullptr;
    // pinned host staging for pointer tables and pair states
    const float** h_tgt = nullptr;
    const float** h_src = nullptr;
    float** h_phi = nullptr;
    float** h_warped = nullptr;
    PairState* h_st = nullptr;
    int h_cap = 0;
    PairState* h_states = nullptr;  // per-call pair states (all chunks)
    int h_states_cap = 0;
    // host-buffer pipeline: H2D / D2H copy streams and per-slot events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_graph[2] = {nullptr, nullptr}, ev_h2d[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr},
                ev_tab[2] = {nullptr, nullptr};

    void ensure_host(int P) {  // pointer tables: two slots of P entries
        if (P <= h_cap) return;
        free_host();
        CK(cudaMallocHost((void**)&h_tgt, sizeof(void*) * 2 * P));
        CK(cudaMallocHost((void**)&h_src, sizeof(void*) * 2 * P));
        CK(cudaMallocHost((void**)&h_phi, sizeof(void*) * 2 * P));
        CK(cudaMallocHost((void**)&h_warped, sizeof(void*) * 2 * P));
        CK(cudaMallocHost((void**)&h_st, sizeof(PairState) * P));
        h_cap = P;
    }
    void ensure_states(int n) {
        if (n <= h_states_cap) return;
        if (h_states) cudaFreeHost(h_states);
        h_states = nullptr;
        CK(cudaMallocHost((void**)&h_states, sizeof(PairState) * n));
        h_states_cap = n;
    }
    void ensure_pipeline() {
        if (h2d) return;
        CK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&ev_graph[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_h2d[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_d2h[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_tab[i], cudaEventDisableTiming));
        }
    }
    void free_pipeline() {
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t* e : {&ev_graph[i], &ev_h2d[i], &ev_d2h[i], &ev_tab[i]})
                if (*e) {
                    cudaEventDestroy(*e);
                    *e = nullptr;
                }
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        h2d = d2h = nullptr;
        if (h_states) cudaFreeHost(h_states);
        h_states = nullptr;
        h_states_cap = 0;
    }
    void free_host() {
        if (h_tgt) cudaFreeHost(h_tgt);
        if (h_src) cudaFreeHost(h_src);
        if (h_phi) cudaFreeHost(h_phi);
        if (h_warped) cudaFreeHost(h_warped);
        if (h_st) cudaFreeHost(h_st);
        h_tgt = h_src = nullptr;
        h_phi = h_warped = nullptr;
        h_st = nullptr;
        h_cap = 0;
    }

    // Workspace for grid d with capacity >= pairs; keeps at most 6 grids, never
    // evicting the ones listed in `keep` (the levels of the call in progress).
    Workspace& workspace(dreg_dims3 d, int pairs, const std::vector<dreg_dims3>& keep = {}) {
        const auto key = std::make_tuple(d.x, d.y, d.z);
        auto it = wss.find(key);
        if (it == wss.end() || it->second->P < pairs) {
            CK(cudaStreamSynchronize(stream));
            if (it != wss.end()) wss.erase(it);
            while (wss.size() >= 6) {
                auto victim = wss.end();
                for (auto jt = wss.begin(); jt != wss.end(); ++jt) {
                    bool kept = false;
                    for (const auto& k : keep)
                        kept |= std::make_tuple(k.x, k.y, k.z) == jt->first;
                    if (!kept && jt->second.get() != last) victim = jt;
                }
                if (victim == wss.end()) break;
                wss.erase(victim);
            }
            auto w = std::make_unique<Workspace>();
            w->alloc(d, pairs);
            it = wss.emplace(key, std::move(w)).first;
        }
        last = it->second.get();
        last->st_shared = nullptr;
        return *last;
    }
};

namespace {

int fail(dreg_cuda_ctx* c, int code, const std::string& m) {
    if (c) c->err = m;
    return code;
}

template <class F>
int guarded(dreg_cuda_ctx* c, F&& f) {
    if (!c) return DREG_INVALID_ARGUMENT;
    try {
        CK(cudaSetDevice(c->device));
        const int r = f();
        if (r == DREG_OK) c->err.clear();
        return r;
    } catch (const ArgFail& e) {
        return fail(c, DREG_INVALID_ARGUMENT, e.msg);
    } catch (const NumFail& e) {
        return fail(c, DREG_NUMERIC, e.msg);
    } catch (const CudaFail& e) {
        return fail(c, DREG_RUNTIME, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(c, DREG_RUNTIME, "host allocation failed");
    }
}

void check_solver(const dreg_solver_cfg* s) {
    if (!s) throw ArgFail("solver config is null");
    const int r = dreg_validate_solver_cfg(s);
    if (r != DREG_OK) {
        if (s->data_term != 1 && s->data_term != 2) throw ArgFail("solver: data term exponent must be 1 or 2");
        if (s->order < 1 || s->order > 6) throw ArgFail("solver: regulariser order must be in [1, 6]");
        if (!(s->lambda >= 0.0)) throw ArgFail("solver: lambda must be >= 0");
        if (!(s->theta > 0.0)) throw ArgFail("solver: theta must be > 0");
        if (!(s->epsilon > 0.0)) throw ArgFail("solver: epsilon must be > 0");
        if (s->max_iters < 1) throw ArgFail("solver: max_iters must be >= 1");
        throw ArgFail("solver: tol must be >= 0");
    }
}

// volume.cpp:15-22 (check_geometry): containers reject non-positive spacing.  The
// registration itself works in voxel units (volume.hpp:25-26), so spacing is only
// validated, like the reference's ScalarVolume constructor does.
void check_spacing(dreg_spacing3 s) {
    if (!(s.x > 0.0) || !(s.y > 0.0) || !(s.z > 0.0)) throw ArgFail("voxel spacing must be positive");
}

void check_dims(dreg_dims3 d, int min_extent, const char* what) {
    if (d.x < 1 || d.y < 1 || d.z < 1) throw ArgFail("volume dims must be positive");
    if (d.x < min_extent || d.y < min_extent || d.z < min_extent)
        throw ArgFail(std::string(what) + ": every axis must have size >= " + std::to_string(min_extent));
}

SolverParams solver_params(const dreg_solver_cfg& s) {
    SolverParams sp{};
    sp.theta = s.theta;
    sp.epsilon = s.epsilon;
    sp.lambda = s.lambda;
    sp.tol = s.tol;
    sp.data_term = s.data_term;
    sp.order = s.order;
    sp.log_objective = s.log_objective;
    sp.accelerate = s.accelerate;
    return sp;
}

// Nesterov coefficients c_k = (alpha_k - 1) / alpha_{k+1}, alpha_0 = 1
// (admm.cpp:198-200, :294-295).  Data-independent, so precomputed.
std::vector<double> nesterov_coefs(int iters, bool accelerate) {
    std::vector<double> c(std::max(iters, 1), 0.0);
    double alpha = 1.0;
    for (int k = 0; k < iters; ++k) {
        const double next = dreg_nesterov_next_alpha(alpha);
        c[k] = accelerate ? (alpha - 1.0) / next : 0.0;
        alpha = next;
    }
    return c;
}

struct Launcher {
    dreg_cuda_ctx* c;
    int count = 0;
    void operator()(cudaError_t e, int kernels = 1) {
        if (e != cudaSuccess) throw CudaFail(std::string("kernel launch: ") + cudaGetErrorString(e));
        count += kernels;
    }
};

XArgs make_xargs(const Workspace& w, const SolverParams& sp, bool diag, bool precise = false) {
    XArgs a{};
    a.precise = precise ? 1 : 0;
    a.twx64 = w.geo.twx64.p;
    a.xtw64 = w.geo.xtw64.p;
    a.F = w.fields(diag);
    a.px = w.geo.px;
    a.twx = w.geo.twx.p;
    a.xtw = w.geo.xtw.p;
    a.xpos = w.geo.xpos.p;
    a.sp = sp;
    a.TL = w.geo.TL;
    a.PM = w.geo.PM;
    a.odd = w.geo.odd;
    a.vec = w.geo.xvec;
    a.prefetch = w.geo.prefetch && (w.geo.M % 4 == 0);
#ifdef DREG_EXPERIMENTS
    a.dbg_skip = env_int("DREG_DBG_SKIP", 0);
#endif
    a.f64 = env_int("DREG_F64", 0);
    a.minb = env_int("DREG_XMINB", 3);
    a.fast_x = env_int("DREG_FAST_X", 1);
    a.fx_variant = env_int("DREG_FX", 22);
    a.pipe = env_int("DREG_PIPE", 1);
    a.pipe_all = env_int("DREG_PIPE_ALL", 0);
    a.pipe_ss = env_int("DREG_PIPE_SS", 1120444);
    a.pipe256 = env_int("DREG_PIPE256", 1);
    if (precise) a.TL = w.geo.TLp;
    a.fd_lines.init((unsigned)(3 * a.TL));
    return a;
}

PArgs make_pargs(const Workspace& w, const SolverParams& sp, bool diag, bool precise = false) {
    PArgs p{};
    p.precise = precise ? 1 : 0;
    p.twy64 = w.geo.twy64.p;
    p.twz64 = w.geo.twz64.p;
    p.sx64 = w.geo.sx64.p;
    p.sy64 = w.geo.sy64.p;
    p.sz64 = w.geo.sz64.p;
    p.lambda64 = sp.lambda;
    p.theta64 = sp.theta;
    p.scale64 = sp.theta / (double)w.geo.N;
    p.cx64 = w.geo.cx64.p;
    p.cy64 = w.geo.cy64.p;
    p.cz64 = w.geo.cz64.p;
    p.cy64_fast = w.geo.cy64_fast.p;
    p.cz64_fast = w.geo.cz64_fast.p;
    p.inv_count = 1.0 / (double)w.geo.N;
    p.F = w.fields(diag);
    p.py = w.geo.py;
    p.pz = w.geo.pz;
    p.twy = w.geo.twy.p;
    p.twz = w.geo.twz.p;
    p.sx = w.geo.sx.p;
    p.sy = w.geo.sy.p;
    p.sz = w.geo.sz.p;
    p.lambda = (float)sp.lambda;
    p.theta = (float)sp.theta;
    p.scale = (float)(sp.theta / (double)w.geo.N);
    p.lam_n = (float)(sp.lambda * (double)w.geo.N / sp.theta);
    p.n_f = (float)w.geo.N;
    // plane_reg_kernel L2-prefetches the plane one wave of resident CTAs ahead (-2% time;
    // an L2 prefetch of the x-pass state instead thrashed L2: +38%)
    p.pf_ahead = env_int("DREG_PLANE_PF", 1);
    p.ss_variant = env_int("DREG_PLANE_SS", 0);
    p.cluster = env_int("DREG_CLUSTER", 1);  // 1: register-blocked cluster kernel where it applies; 2: generic; 0: split
    p.ss_prefetch = env_int("DREG_PLANE_UPF", 1);
    p.ss_stream = env_int("DREG_PLANE_STREAM", 1);
    p.order = sp.order;
    p.PY = w.geo.PY;
    p.energy_out = w.energy.p;
    p.sy_fast = w.geo.sy_fast.p;
    p.sz_fast = w.geo.sz_fast.p;
    p.fast = precise ? 0 : w.geo.fast;
    p.fd_ny.init((unsigned)w.geo.Ny);
    p.fd_nz.init((unsigned)w.geo.Nz);
    return p;
}

// Precision policy: 0 auto -- fp64 spectral arithmetic and storage for
// solves over 100 iterations (the accelerated iteration amplifies rounding) and for the
// l1 data term (its shrinkage branch does); 1 always fp32; 2 always fp64.
bool solve_precise(int policy, const dreg_solver_cfg& s) {
    return policy == 2 || (policy == 0 && (s.max_iters > 100 || s.data_term == 1));
}

// Which solves run the spectral-state iteration (plane_fast.cuh MODE 2 + X_SS): l2, fp32,
// grids the register-blocked plane kernel and the pipelined x-pass cover, no diagnostics.
bool solve_uses_spectral_state(const Workspace& w, const dreg_solver_cfg& s, const XArgs& xa, bool diag, bool need_tail,
                               bool precise) {
    return !diag && !need_tail && !precise && s.data_term == 2 && w.geo.fast >= 2 &&
           plane_reg_supported(w.geo.Ny, w.geo.Nz) && xpass_ss_eligible(xa) && env_int("DREG_SS", 1) != 0;
}
bool ss_needs_change(const dreg_solver_cfg& s) { return s.tol > 0.0 || env_int("DREG_SS_CHG", 0) != 0; }

// One accelerated-ADMM velocity solve for all active pairs (admm.cpp:252-314):
// grad/diff setup, then I iterations of (plane, xpass).  need_tail adds the last
// w-update (only the constraint-residual diagnostic depends on it).
void enqueue_solve(Launcher& L, Workspace& w, int P, const dreg_solver_cfg& s, bool diag, bool need_tail,
                   bool with_setup, cudaStream_t st) {
    const bool log_obj = diag && s.log_objective;
    SolverParams sp = solver_params(s);
    sp.log_objective = log_obj ? 1 : 0;
    const int I = s.max_iters;
    const std::vector<double> coef = nesterov_coefs(I, s.accelerate != 0);

    // precision policy: the accelerated iteration amplifies per-iteration
    // rounding, so long solves get fp64 spectral arithmetic (storage stays fp32)
    const bool precise = solve_precise(L.c->precision, s);
    if (precise && !w.S64.p) throw ArgFail("precise solve needs the workspace's fp64 spectrum");
    // the exact fp64 point-wise form (l1, precise) reads warped and target themselves
    if (with_setup) L(launch_grad_diff(w.vg(), w.regbufs(), w.fields(diag), s.data_term == 1 || precise, P, st));
    XArgs xa = make_xargs(w, sp, diag, precise);
    PArgs pa = make_pargs(w, sp, diag, precise);
    pa.need_tail = need_tail ? 1 : 0;
    if (log_obj && !w.S2.p) throw ArgFail("log_objective needs the workspace's scratch spectrum");
    auto energy = [&](int k) {
        // objective_k = data term + lambda * spectral_energy(v_k)   (admm.cpp:288-292):
        // r2c(v_k) goes to the scratch spectrum S2, so the iteration's own spectrum S is
        // never touched and v does not depend on log_objective
        XArgs fa = xa;
        fa.k = k;
        fa.add_bh = 0;
        fa.F.S = w.S2.p;
        fa.F.S64 = w.S264.p;
        PArgs ea = pa;
        ea.k = k;
        ea.F.S = w.S2.p;
        ea.F.S64 = w.S264.p;
        L(launch_xpass(fa, X_FWD, P, st));
        L(launch_plane(ea, 1, P, st));
        L(launch_objective_accumulate(w.fields(true), w.energy.p, sp.lambda, k, P, st));
    };
    xa.k = 0;
    xa.coef = 0.0;
    xa.coef_prev = 0.0;
    L(launch_xpass(xa, X_FIRST, P, st));
    if (log_obj) energy(0);
    // Spectral-state iteration (plane_fast.cuh MODE 2 + X_SS): the ADMM state is kept as two
    // Fourier-domain iterates U_j, U_{j-1} inside the plane pass, the x-pass streams only
    // v, grad and diff.  Same recurrence (admm.cpp:275-308) in fp32; not for the logged /
    // diagnostic solves (no w, b fields to take the residual from), l1 or precise mode.
    const bool ss = solve_uses_spectral_state(w, s, xa, diag, need_tail, precise);
    if (ss) {
        // without a tolerance the change norm is not needed: v is neither read nor written
        // until the last iteration (an exactly-zero change is still caught at k = 0)
        const int xmode = ss_needs_change(s) ? X_SS : X_SSN;
        float2* const ubuf[2] = {reinterpret_cast<float2*>(w.BH.p), reinterpret_cast<float2*>(w.BP.p)};
        pa.inv_nf = (float)(1.0 / (double)w.geo.N);
        for (int k = 1; k < I; ++k) {
            pa.k = k - 1;
            pa.c_cur = (float)coef[k - 1];
            pa.c_prev = k >= 2 ? (float)coef[k - 2] : 0.f;
            pa.has1 = k >= 2;
            pa.has0 = pa.c_prev != 0.f;
            pa.U1 = ubuf[(k - 1) & 1];
            pa.U0 = ubuf[k & 1];
            L(launch_plane(pa, 2, P, st));
            xa.k = k;
            xa.ss_last = k == I - 1;
            L(launch_xpass(xa, xmode, P, st));
        }
        return;
    }
    // The dual iterates ping-pong between the two b buffers: pass k reads b_{k-1} (F.BP) and
    // b_{k-2} (F.BH), re-forms b_hat_{k-1} with c_{k-2} and writes b_k over b_{k-2}.
    float* const bbuf[2] = {xa.F.BH, xa.F.BP};
    for (int k = 1; k < I; ++k) {
        pa.k = k - 1;
        L(launch_plane(pa, 0, P, st));
        xa.k = k;
        xa.coef = coef[k - 1];
        xa.coef_prev = k >= 2 ? coef[k - 2] : 0.0;
        xa.F.BP = bbuf[(k - 1) & 1];
        xa.F.BH = bbuf[k & 1];
        L(launch_xpass(xa, k == 1 ? X_SECOND : X_GENERAL, P, st));
        if (log_obj) energy(k);
    }
    if (need_tail) {
        pa.k = I - 1;
        L(launch_plane(pa, 0, P, st));
        xa.k = I;
        L(launch_xpass(xa, X_TAIL, P, st));
    }
}

// register_pair (registration.cpp:180-283) for all pairs of the chunk; lv holds the
// level workspaces coarsest first, the finest (original grid) last.  Per-pair state
// lives in the finest workspace and is shared by every level.
void smooth_or_copy(Launcher& L, const Workspace& w, int P, bool smooth, cudaStream_t st) {
    const VolGeom g = w.vg();
    const RegBuffers R = w.regbufs();
    if (smooth) {  // binomial_smooth = x, y, z passes (registration.cpp:141-143)
        L(launch_smooth_axis(g, R.tmpA, R.I0, 0, P, st));
        L(launch_smooth_axis(g, R.I0, R.tmpA, 1, P, st));
        L(launch_smooth_axis(g, R.tmpA, R.I0, 2, P, st));
        L(launch_smooth_axis(g, R.tmpB, R.I1, 0, P, st));
        L(launch_smooth_axis(g, R.I1, R.tmpB, 1, P, st));
        L(launch_smooth_axis(g, R.tmpB, R.I1, 2, P, st));
    } else {
        CK(cudaMemcpyAsync(R.I0, R.tmpA, sizeof(float) * g.N * P, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(R.I1, R.tmpB, sizeof(float) * g.N * P, cudaMemcpyDeviceToDevice, st));
    }
}

void enqueue_registration(Launcher& L, const std::vector<Workspace*>& lv, int P, const dreg_reg_cfg& cfg,
                          cudaStream_t st) {
    const int Lv = (int)lv.size();
    Workspace& fine = *lv.back();
    for (Workspace* w : lv) w->st_shared = (w == &fine) ? nullptr : fine.st.p;
    const RegBuffers Rf = fine.regbufs();
    const Fields Ff = fine.fields(false);
    // normalise with one shared range (registration.cpp:205), pyramid (:208-214), smoothing (:216-221)
    L(launch_prep_normalize(fine.vg(), Rf, Ff, P, st), 3);
    for (int l = Lv - 1; l > 0; --l) {
        const RegBuffers a = lv[l]->regbufs(), b = lv[l - 1]->regbufs();
        L(launch_pyr_down(lv[l]->vg(), lv[l - 1]->vg(), a.tmpA, a.tmpB, b.tmpA, b.tmpB, P, st));
    }
    for (int l = 0; l < Lv; ++l) smooth_or_copy(L, *lv[l], P, cfg.smooth_levels != 0, st);
    dreg_solver_cfg s = cfg.solver;
    for (int l = 0; l < Lv; ++l) {
        Workspace& w = *lv[l];
        const VolGeom g = w.vg();
        const RegBuffers R = w.regbufs();
        const Fields F = w.fields(false);
        if (l == 0) L(launch_level_init(g, R, F, 0, P, st));
        else L(launch_level_up(lv[l - 1]->vg(), g, lv[l - 1]->regbufs(), R, F, l, P, st));
        s.max_iters = cfg.max_admm_iters_per_level[l];
        const int K = std::max(0, cfg.max_warps_per_level[l]);
        for (int wi = 0; wi < K; ++wi) {
            enqueue_solve(L, w, P, s, false, false, true, st);
            L(launch_compose_decide(g, R, F, cfg.warp_improvement_threshold, K, P, st));
        }
    }
    L(launch_finalize(fine.vg(), Rf, Ff, P, st));
}

std::string graph_key(int P, const dreg_reg_cfg& c, const std::vector<Workspace*>& lv) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%d|%d|%d|%.17g|%.17g|%.17g|%.17g|%d|%.17g|%d|%d", P, c.solver.data_term,
                  c.solver.order, c.solver.lambda, c.solver.theta, c.solver.epsilon, c.solver.tol, c.solver.accelerate,
                  c.warp_improvement_threshold, c.smooth_levels, c.levels);
    std::string k = buf;
    for (int l = 0; l < c.levels; ++l)
        k += "|" + std::to_string(c.max_warps_per_level[l]) + "x" + std::to_string(c.max_admm_iters_per_level[l]) +
             "@" + std::to_string(lv[l]->id);
    return k;
}

// L2 residency of the x-spectrum (DREG_L2_PERSIST = set-aside MB, 0 = off): every
// kernel node of the registration graph gets an access-policy window over S with
// hitProp persisting, so the spectrum written by one pass stays in L2 for the next
// while the ADMM state streams past it.  Only pays when the chunk's spectrum
// (3 * 2(M/2+1)/M * 4 B/voxel per pair) fits the set-aside.
void apply_l2_window(dreg_cuda_ctx* c, Workspace& w, cudaGraph_t graph) {
    const int mb = env_int("DREG_L2_PERSIST", 0);
    if (mb <= 0) return;
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, c->device));
    const size_t want = std::min((size_t)mb << 20, (size_t)prop.persistingL2CacheMaxSize);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    const size_t bytes = std::min(sizeof(float2) * w.S.n, (size_t)prop.accessPolicyMaxWindowSize);
    cudaKernelNodeAttrValue v{};
    v.accessPolicyWindow.base_ptr = w.S.p;
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)want / (double)bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    size_t n = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(graph, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t == cudaGraphNodeTypeKernel)
            CK(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v));
    }
    if (env_int("DREG_L2_VERBOSE", 0))
        std::fprintf(stderr, "[dreg] L2 persist: set-aside %zu MB (max %zu MB), window %zu MB (max %zu MB), hit %.3f\n",
                     want >> 20, (size_t)prop.persistingL2CacheMaxSize >> 20, bytes >> 20,
                     (size_t)prop.accessPolicyMaxWindowSize >> 20, v.accessPolicyWindow.hitRatio);
}

void run_registration(dreg_cuda_ctx* c, const std::vector<Workspace*>& lv, int P, const dreg_reg_cfg& cfg) {
    cudaStream_t st = c->stream;
    Workspace& w = *lv.back();
    if (!c->use_graphs) {
        Launcher L{c};
        enqueue_registration(L, lv, P, cfg, st);
        c->launches += L.count;
        return;
    }
    const std::string key = graph_key(P, cfg, lv) + "|prec" + std::to_string(c->precision);
    auto it = w.graphs.find(key);
    if (it == w.graphs.end()) {
        Launcher L{c};
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_registration(L, lv, P, cfg, st);
        } catch (...) {
            cudaStreamEndCapture(st, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        CK(cudaStreamEndCapture(st, &graph));
        apply_l2_window(c, w, graph);
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(e);
        it = w.graphs.emplace(key, std::make_pair(exec, L.count)).first;
    }
    CK(cudaGraphLaunch(it->second.first, st));
    c->launches += it->second.second;
}

// registration.cpp:182-198, in the reference's order.  Per-level ADMM caps are checked
// only on levels that run a solve (the reference validates them inside solve_velocity);
// a negative warp cap runs no warps, like the reference's `warp < max_warps` loop.
void validate_reg(const dreg_reg_cfg* cfg, dreg_dims3 d) {
    if (!cfg) throw ArgFail("registration config is null");
    check_solver(&cfg->solver);
    if (cfg->levels < 1) throw ArgFail("register_pair: levels must be >= 1");
    if (!(cfg->warp_improvement_threshold > 0.0 && cfg->warp_improvement_threshold < 1.0))
        throw ArgFail("register_pair: warp improvement threshold must be in (0,1)");
    if (d.x < 1 || d.y < 1 || d.z < 1) throw ArgFail("volume dims must be positive");
    const long long min_extent = cfg->levels > 40 ? (1LL << 42) : (4LL << (cfg->levels - 1));
    if (d.x < min_extent || d.y < min_extent || d.z < min_extent)
        throw ArgFail("register_pair: dims too small for the level count");
    if (cfg->levels > DREG_MAX_LEVELS)
        throw ArgFail("register_pair: more than " + std::to_string(DREG_MAX_LEVELS) + " levels (axes >= " +
                      std::to_string(4 << (DREG_MAX_LEVELS - 1)) + " voxels) exceed one device");
    for (int l = 0; l < cfg->levels; ++l) {
        if (cfg->max_warps_per_level[l] > DREG_MAX_WARPS)
            throw ArgFail("register_pair: warp cap above " + std::to_string(DREG_MAX_WARPS) +
                          " (per-level log capacity, dreg_cuda.h)");
        if (cfg->max_warps_per_level[l] >= 1 && cfg->max_admm_iters_per_level[l] < 1)
            throw ArgFail("solver: max_iters must be >= 1");
    }
}

void fill_results(const PairState* hs, int P, const std::vector<dreg_dims3>& dl, dreg_pair_result* out,
                  double elapsed) {
    for (int p = 0; p < P; ++p) {
        dreg_pair_result& r = out[p];
        std::memset(&r, 0, sizeof r);
        const PairState& s = hs[p];
        r.status = s.status;
        r.velocity_count = s.velocity_count;
        r.solves = s.solves;
        r.levels = (int)dl.size();
        for (int l = 0; l < r.levels; ++l) {
            dreg_level_log& lg = r.per_level[l];
            lg.dims = dl[l];
            lg.warps = s.level_warps[l];
            for (int i = 0; i <= lg.warps && i <= DREG_MAX_WARPS; ++i) lg.mean_sad[i] = s.mean_sad[l][i];
            for (int i = 0; i < lg.warps && i < DREG_MAX_WARPS; ++i) lg.solver_iterations[i] = s.solver_iterations[l][i];
        }
        r.elapsed_seconds = elapsed;
        r.folding_voxels = (int64_t)s.folding;
        r.min_det = s.min_det;
    }
}

// Pairs per device launch (automatic unless dreg_cuda_set_batch_chunk).  Host-buffer
// batches use 64-pair chunks so one chunk's H2D / D2H overlaps the next chunk's
// registration; device-resident batches have no copies to hide and take up to 256
// pairs per launch, which keeps the persistent x-pass's per-CTA tile ranges long
// (measured at 128 config-3 pairs: 64 -> 112.9, 128 -> 115.1 registrations/s).
int pick_chunk(dreg_cuda_ctx* c, dreg_dims3 d, int n_pairs, bool host, bool precise) {
    if (c->chunk > 0) return std::min(c->chunk, n_pairs);
    Geometry tmp;
    tmp.M = d.x;
    tmp.Ny = d.y;
    tmp.Nz = d.z;
    tmp.hx = d.x / 2 + 1;
    tmp.N = (long long)d.x * d.y * d.z;
    tmp.lines = (long long)d.y * d.z;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t per = Workspace::bytes_per_pair(tmp, host) + (precise ? sizeof(double2) * 3 * (size_t)tmp.hx * tmp.lines : 0);
    size_t fit = (size_t)(0.6 * (double)free_b) / std::max<size_t>(per, 1);
    {
        auto it = c->wss.find(std::make_tuple(d.x, d.y, d.z));
        if (it != c->wss.end()) fit = std::max<size_t>(fit, (size_t)it->second->P);
    }
    int P = (int)std::min<size_t>(fit, host ? 64 : 256);
    return std::max(1, std::min(P, n_pairs));
}

// DREG_GUARD: verify every workspace buffer's guard bands (see DevArray)
void check_guards(dreg_cuda_ctx* c) {
    if (!guard_mode()) return;
    CK(cudaDeviceSynchronize());
    for (auto& kv : c->wss)
        if (const char* b = kv.second->corrupted_buffer())
            throw CudaFail(std::string("guard band corrupted after the call: buffer ") + b + " of workspace " +
                           std::to_string(std::get<0>(kv.first)) + "x" + std::to_string(std::get<1>(kv.first)) + "x" +
                           std::to_string(std::get<2>(kv.first)));
}

}  // namespace

// =================================== C ABI ======================================
extern "C" {

void dreg_solver_cfg_default(dreg_solver_cfg* c) {
    if (!c) return;
    c->data_term = 1;
    c->order = 2;
    c->lambda = 0.0;
    c->theta = 0.1;
    c->epsilon = 1e-6;
    c->max_iters = 100;
    c->tol = 0.0;
    c->accelerate = 1;
    c->log_objective = 1;
}

int dreg_validate_solver_cfg(const dreg_solver_cfg* c) {
    if (!c) return DREG_INVALID_ARGUMENT;
    if (c->data_term != 1 && c->data_term != 2) return DREG_INVALID_ARGUMENT;
    if (c->order < 1 || c->order > 6) return DREG_INVALID_ARGUMENT;
    if (!(c->lambda >= 0.0)) return DREG_INVALID_ARGUMENT;
    if (!(c->theta > 0.0)) return DREG_INVALID_ARGUMENT;
    if (!(c->epsilon > 0.0)) return DREG_INVALID_ARGUMENT;
    if (c->max_iters < 1) return DREG_INVALID_ARGUMENT;
    if (!(c->tol >= 0.0)) return DREG_INVALID_ARGUMENT;
    return DREG_OK;
}

int dreg_make_registration_config(int profile, const dreg_solver_cfg* solver, int levels, dreg_reg_cfg* out) {
    if (!solver || !out || levels < 1 || levels > DREG_MAX_LEVELS) return DREG_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof *out);
    out->solver = *solver;
    out->levels = levels;
    out->profile = profile;
    out->warp_improvement_threshold = 0.02;
    out->smooth_levels = 1;
    if (profile == DREG_PROFILE_CAPPED) {
        for (int l = 0; l < levels; ++l) {
            out->max_admm_iters_per_level[l] = 5;
            out->max_warps_per_level[l] = 10;
        }
        out->max_admm_iters_per_level[0] = 10;
        out->max_warps_per_level[levels - 1] = 5;
    } else {
        for (int l = 0; l < levels; ++l) {
            out->max_admm_iters_per_level[l] = 200;
            out->max_warps_per_level[l] = 50;
        }
        if (out->solver.tol <= 0.0) out->solver.tol = 0.01;
    }
    return DREG_OK;
}

double dreg_nesterov_next_alpha(double alpha) { return 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * alpha * alpha)); }

int dreg_laplacian_symbol(int order, dreg_dims3 d, double* out) {
    if (order < 1 || order > 6 || d.x < 2 || d.y < 2 || d.z < 2 || !out) return DREG_INVALID_ARGUMENT;
    std::vector<double> cx(d.x), cy(d.y), cz(d.z);
    for (int k = 0; k < d.x; ++k) cx[k] = std::cos(2.0 * kPi * k / d.x);
    for (int k = 0; k < d.y; ++k) cy[k] = std::cos(2.0 * kPi * k / d.y);
    for (int k = 0; k < d.z; ++k) cz[k] = std::cos(2.0 * kPi * k / d.z);
    cx[0] = cy[0] = cz[0] = 1.0;
    size_t i = 0;
    for (int r = 0; r < d.z; ++r)
        for (int q = 0; q < d.y; ++q) {
            const double yz = 3.0 - cy[q] - cz[r];
            for (int p = 0; p < d.x; ++p, ++i) {
                const double base = 2.0 * (yz - cx[p]);
                double v = base;
                for (int e = 1; e < order; ++e) v *= base;
                out[i] = v;
            }
        }
    return DREG_OK;
}

int dreg_cuda_ctx_create(int device, dreg_cuda_ctx** out) {
    if (!out) return DREG_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return DREG_RUNTIME;
    if (device < 0 || device >= n) return DREG_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return DREG_RUNTIME;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DREG_RUNTIME;
    if (prop.major < 10) return DREG_RUNTIME;  // sm_100a binary only
    auto* c = new dreg_cuda_ctx();
    c->device = device;
    if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return DREG_RUNTIME;
    }
    c->stream = c->own;
    *out = c;
    return DREG_OK;
}

void dreg_cuda_ctx_destroy(dreg_cuda_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->h2d) cudaStreamSynchronize(c->h2d);
    if (c->d2h) cudaStreamSynchronize(c->d2h);
    c->wss.clear();
    c->last = nullptr;
    c->free_host();
    c->free_pipeline();
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
}

const char* dreg_cuda_last_error(const dreg_cuda_ctx* c) { return c ? c->err.c_str() : "null context"; }

int dreg_cuda_set_stream(dreg_cuda_ctx* c, void* stream) {
    if (!c) return DREG_INVALID_ARGUMENT;
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
    return DREG_OK;
}

int64_t dreg_cuda_kernel_launches(const dreg_cuda_ctx* c) { return c ? c->launches : 0; }

int dreg_cuda_set_batch_chunk(dreg_cuda_ctx* c, int pairs) {
    if (!c || pairs < 0) return DREG_INVALID_ARGUMENT;
    c->chunk = pairs;
    return DREG_OK;
}

int dreg_cuda_set_precision(dreg_cuda_ctx* c, int mode) {
    if (!c || mode < 0 || mode > 2) return DREG_INVALID_ARGUMENT;
    c->precision = mode;
    return DREG_OK;
}

int dreg_cuda_set_use_graphs(dreg_cuda_ctx* c, int enable) {
    if (!c) return DREG_INVALID_ARGUMENT;
    c->use_graphs = enable ? 1 : 0;
    return DREG_OK;
}

static int register_impl(dreg_cuda_ctx* c, int n_pairs, const float* const* tgt_host, const float* const* src_host,
                         const float* tgt_dev, const float* src_dev, dreg_dims3 d, const dreg_reg_cfg* cfg,
                         float* const* phi_host, float* const* warped_host, float* phi_dev, float* warped_dev,
                         dreg_pair_result* results, dreg_pair_record* rec_dev = nullptr, int pair_base = 0,
                         int device_tag = 0) {
    const auto t0 = std::chrono::steady_clock::now();
    if (n_pairs < 0) throw ArgFail("n_pairs must be >= 0");
    validate_reg(cfg, d);
    if (n_pairs == 0) return DREG_OK;
    const bool host = tgt_host != nullptr;
    // Host buffers spanning several chunks: chunk j+1's H2D and chunk j-1's D2H overlap
    // chunk j's registration (copy streams + double-buffered staging).  A single chunk
    // is not split for overlap: measured at 32 config-2 pairs, 2 x 16 ran 2% slower
    // end to end than 1 x 32 (tools/e2e_probe.py).
    bool precise_any = false;
    {
        dreg_solver_cfg s = cfg->solver;
        for (int l = 0; l < cfg->levels; ++l) {
            s.max_iters = cfg->max_admm_iters_per_level[l];
            precise_any |= cfg->max_warps_per_level[l] > 0 && solve_precise(c->precision, s);
        }
    }
    const int chunk = pick_chunk(c, d, n_pairs, host, precise_any);
    // level grids, coarsest first (registration.cpp:208-214: dims halved, rounded up)
    std::vector<dreg_dims3> dl((size_t)cfg->levels);
    dl.back() = d;
    for (int l = cfg->levels - 1; l > 0; --l)
        dl[l - 1] = {(dl[l].x + 1) / 2, (dl[l].y + 1) / 2, (dl[l].z + 1) / 2};
    std::vector<Workspace*> lv((size_t)cfg->levels);
    for (int l = 0; l < cfg->levels; ++l) lv[l] = &c->workspace(dl[l], chunk, dl);
    Workspace& w = c->workspace(d, chunk, dl);
    lv.back() = &w;
    {  // fp64 spectra for the levels whose solves run in precise mode (before graph capture)
        dreg_solver_cfg s = cfg->solver;
        for (int l = 0; l < cfg->levels; ++l) {
            s.max_iters = cfg->max_admm_iters_per_level[l];
            if (cfg->max_warps_per_level[l] > 0 && solve_precise(c->precision, s)) lv[l]->ensure_s64();
        }
    }
    c->ensure_host(w.P);
    c->ensure_states(n_pairs);
    if (tgt_host) w.ensure_staging();
    const size_t N = (size_t)w.geo.N;
    const size_t Pc = (size_t)w.P;
    cudaStream_t st = c->stream;
    int first_bad = DREG_OK;
    const int nchunks = (n_pairs + chunk - 1) / chunk;
    if (host) {
        c->ensure_pipeline();
        for (int q = 0; q < n_pairs; ++q)
            if (!tgt_host[q] || !src_host[q]) throw ArgFail("null input volume");
        // stage slots are free once the previous chunk's registration on st has consumed them
        CK(cudaEventRecord(c->ev_graph[0], st));
        CK(cudaEventRecord(c->ev_graph[1], st));
        CK(cudaEventRecord(c->ev_d2h[0], st));
        CK(cudaEventRecord(c->ev_d2h[1], st));
    }
    // H2D of chunk j's inputs into stage slot j % 2 (h2d stream)
    auto issue_h2d = [&](int j) {
        const int slot = j & 1, p0 = j * chunk, P = std::min(chunk, n_pairs - p0);
        CK(cudaStreamWaitEvent(c->h2d, c->ev_graph[slot], 0));  // chunk j-2 done with the slot
        for (int p = 0; p < P; ++p) {
            CK(cudaMemcpyAsync(w.stage_t.p + (slot * Pc + p) * N, tgt_host[p0 + p], sizeof(float) * N,
                               cudaMemcpyHostToDevice, c->h2d));
            CK(cudaMemcpyAsync(w.stage_s.p + (slot * Pc + p) * N, src_host[p0 + p], sizeof(float) * N,
                               cudaMemcpyHostToDevice, c->h2d));
        }
        CK(cudaEventRecord(c->ev_h2d[slot], c->h2d));
    };
    if (host) issue_h2d(0);
    for (int j = 0; j < nchunks; ++j) {
        const int p0 = j * chunk;
        const int P = std::min(chunk, n_pairs - p0);
        const int slot = host ? (j & 1) : 0;
        if (host && j + 1 < nchunks) issue_h2d(j + 1);  // overlaps this chunk's registration
        // pinned pointer tables: slot reused two chunks later, once its H2D has executed
        if (host) CK(cudaEventSynchronize(c->ev_tab[slot]));
        else CK(cudaStreamSynchronize(st));
        const float** ht = c->h_tgt + slot * Pc;
        const float** hs = c->h_src + slot * Pc;
        float** hp = c->h_phi + slot * Pc;
        float** hw = c->h_warped + slot * Pc;
        for (int p = 0; p < P; ++p) {
            const int q = p0 + p;
            if (host) {
                ht[p] = w.stage_t.p + (slot * Pc + p) * N;
                hs[p] = w.stage_s.p + (slot * Pc + p) * N;
                hp[p] = (phi_host && phi_host[q]) ? w.phi_soa.p + p * 3 * N : nullptr;
                hw[p] = (warped_host && warped_host[q]) ? w.warped.p + (slot * Pc + p) * N : nullptr;
            } else {
                ht[p] = tgt_dev + (size_t)q * N;
                hs[p] = src_dev + (size_t)q * N;
                hp[p] = phi_dev ? phi_dev + (size_t)q * 3 * N : nullptr;
                hw[p] = warped_dev ? warped_dev + (size_t)q * N : nullptr;
            }
        }
        CK(cudaMemcpyAsync(w.tgt_tab.p, ht, sizeof(void*) * P, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(w.src_tab.p, hs, sizeof(void*) * P, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(w.phi_tab.p, hp, sizeof(void*) * P, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(w.warped_tab.p, hw, sizeof(void*) * P, cudaMemcpyHostToDevice, st));
        if (host) {
            CK(cudaEventRecord(c->ev_tab[slot], st));
            CK(cudaStreamWaitEvent(st, c->ev_h2d[slot], 0));  // inputs landed
            CK(cudaStreamWaitEvent(st, c->ev_d2h[slot], 0));  // chunk j-2's outputs left the slot
        }
        run_registration(c, lv, P, *cfg);
        if (rec_dev) {  // per-pair records for the multi-device all-gather
            CK(launch_pack_records(w.st.p, P, pair_base + p0, device_tag, cfg->levels, rec_dev + p0, st));
            c->launches += 1;
        }
        if (host) {
            for (int p = 0; p < P; ++p)
                if (phi_host && phi_host[p0 + p]) {
                    CK(launch_soa_to_aos((long long)N, w.phi_soa.p + p * 3 * N, w.stage3.p + (slot * Pc + p) * 3 * N,
                                         st));
                    c->launches += 1;
                }
        }
        // pair states stay on st (tiny): the next chunk's reset cannot overtake them
        CK(cudaMemcpyAsync(c->h_states + p0, w.st.p, sizeof(PairState) * P, cudaMemcpyDeviceToHost, st));
        if (host) {
            CK(cudaEventRecord(c->ev_graph[slot], st));
            CK(cudaStreamWaitEvent(c->d2h, c->ev_graph[slot], 0));
            for (int p = 0; p < P; ++p) {
                const int q = p0 + p;
                if (phi_host && phi_host[q])
                    CK(cudaMemcpyAsync(phi_host[q], w.stage3.p + (slot * Pc + p) * 3 * N, sizeof(float) * 3 * N,
                                       cudaMemcpyDeviceToHost, c->d2h));
                if (warped_host && warped_host[q])
                    CK(cudaMemcpyAsync(warped_host[q], w.warped.p + (slot * Pc + p) * N, sizeof(float) * N,
                                       cudaMemcpyDeviceToHost, c->d2h));
            }
            CK(cudaEventRecord(c->ev_d2h[slot], c->d2h));
        }
    }
    CK(cudaStreamSynchronize(st));
    if (host) CK(cudaStreamSynchronize(c->d2h));
    check_guards(c);
    std::vector<PairState> states(c->h_states, c->h_states + n_pairs);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int q = 0; q < n_pairs; ++q) {
        if (states[q].status != DREG_OK && first_bad == DREG_OK) first_bad = states[q].status;
    }
    if (results) fill_results(states.data(), n_pairs, dl, results, el);
    if (first_bad != DREG_OK) {
        c->err = "register_pair: non-finite values (input volumes, velocity or deformation)";
        return first_bad;
    }
    return DREG_OK;
}

// Internal (engine_internal.h): host-buffer batch that also writes each pair's
// dreg_pair_record into the device buffer rec_dev (the multi-device gather's send buffer).
int dregb_register_batch_records(dreg_cuda_ctx* c, int n_pairs, const float* const* targets,
                                 const float* const* sources, dreg_dims3 dims, const dreg_reg_cfg* cfg,
                                 float* const* phi_out, float* const* warped_out, dreg_pair_result* results,
                                 dreg_pair_record* rec_dev, int pair_base, int device_tag) {
    return guarded(c, [&] {
        if (n_pairs > 0 && (!targets || !sources)) throw ArgFail("null input arrays");
        return register_impl(c, n_pairs, targets, sources, nullptr, nullptr, dims, cfg, phi_out, warped_out,
                             nullptr, nullptr, results, rec_dev, pair_base, device_tag);
    });
}

int dreg_cuda_register_pair(dreg_cuda_ctx* c, const float* target, const float* source, dreg_dims3 dims,
                            dreg_spacing3 spacing, const dreg_reg_cfg* cfg, float* phi_out, float* warped_out,
                            dreg_pair_result* result) {
    const float* t[1] = {target};
    const float* s[1] = {source};
    float* po[1] = {phi_out};
    float* wo[1] = {warped_out};
    return guarded(c, [&] {
        check_spacing(spacing);
        if (!target || !source) throw ArgFail("null input volume");
        return register_impl(c, 1, t, s, nullptr, nullptr, dims, cfg, po, wo, nullptr, nullptr, result);
    });
}

int dreg_cuda_register_batch(dreg_cuda_ctx* c, int n_pairs, const float* const* targets,
                             const float* const* sources, dreg_dims3 dims, dreg_spacing3 spacing,
                             const dreg_reg_cfg* cfg, float* const* phi_out, float* const* warped_out,
                             dreg_pair_result* results) {
    return guarded(c, [&] {
        check_spacing(spacing);
        if (n_pairs > 0 && (!targets || !sources)) throw ArgFail("null input arrays");
        return register_impl(c, n_pairs, targets, sources, nullptr, nullptr, dims, cfg, phi_out, warped_out,
                             nullptr, nullptr, results);
    });
}

int dreg_cuda_register_batch_device(dreg_cuda_ctx* c, int n_pairs, const float* targets_dev,
                                    const float* sources_dev, dreg_dims3 dims, dreg_spacing3 spacing,
                                    const dreg_reg_cfg* cfg, float* phi_dev_out, float* warped_dev_out,
                                    dreg_pair_result* results) {
    return guarded(c, [&] {
        check_spacing(spacing);
        if (n_pairs > 0 && (!targets_dev || !sources_dev)) throw ArgFail("null input arrays");
        return register_impl(c, n_pairs, nullptr, nullptr, targets_dev, sources_dev, dims, cfg, nullptr, nullptr,
                             phi_dev_out, warped_dev_out, results);
    });
}

// ---- single solve ---------------------------------------------------------------
int dreg_cuda_solve_velocity(dreg_cuda_ctx* c, const float* target, const float* warped_source, dreg_dims3 d,
                             const dreg_solver_cfg* cfg, float* velocity_out, dreg_solver_diag* diag) {
    return guarded(c, [&] {
        check_solver(cfg);
        check_dims(d, 2, "image_gradient");
        if (!target || !warped_source || !velocity_out) throw ArgFail("null buffer");
        Workspace& w = c->workspace(d, 1);
        w.ensure_diag(cfg->max_iters);
        w.ensure_staging();
        if (cfg->log_objective && !w.S2.p) w.S2.alloc(w.S.n);
        if (solve_precise(c->precision, *cfg)) {
            w.ensure_s64();
            if (cfg->log_objective && !w.S264.p) w.S264.alloc(w.S.n);
        }
        const size_t N = (size_t)w.geo.N;
        cudaStream_t st = c->stream;
        Launcher L{c};
        CK(cudaMemcpyAsync(w.I0.p, target, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(w.W0.p, warped_source, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(w.diag.p, 0, sizeof(double) * 3 * w.diag_iters, st));
        L(launch_state_reset(w.st.p, 1, st));
        enqueue_solve(L, w, 1, *cfg, true, true, true, st);
        L(launch_soa_to_aos((long long)N, w.V.p, w.stage3.p, st));
        c->launches += L.count;
        CK(cudaMemcpyAsync(velocity_out, w.stage3.p, sizeof(float) * 3 * N, cudaMemcpyDeviceToHost, st));
        PairState hs;
        CK(cudaMemcpyAsync(&hs, w.st.p, sizeof(PairState), cudaMemcpyDeviceToHost, st));
        std::vector<double> dg((size_t)3 * w.diag_iters);
        CK(cudaMemcpyAsync(dg.data(), w.diag.p, sizeof(double) * dg.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        check_guards(c);
        if (diag) {
            diag->iterations = hs.iterations;
            diag->final_change = hs.final_change;
            diag->converged = hs.solve_done;
            for (int k = 0; k < hs.iterations; ++k) {
                if (diag->constraint_residual) diag->constraint_residual[k] = dg[3 * k + 1];
                if (diag->objective && cfg->log_objective) diag->objective[k] = dg[3 * k + 2];
            }
        }
        for (size_t i = 0; i < 3 * N; ++i)
            if (!std::isfinite(velocity_out[i]))
                throw NumFail("solve_velocity: velocity field contains non-finite values");
        return DREG_OK;
    });
}

// ---- measurement ----------------------------------------------------------------
// CUDA-event timing of one steady-state ADMM iteration (plane + x-pass X_GENERAL) on
// the last workspace, with `s`'s parameters and its precision policy (fp64 spectral
// arithmetic when the policy picks it for s->max_iters).  out: [xpass ms, plane ms,
// x-pass algorithmic bytes, plane algorithmic bytes, pairs, precise].
static int time_iteration_impl(dreg_cuda_ctx* c, const dreg_solver_cfg* scfg, int reps, double* out) {
    if (!c->last) throw ArgFail("time_kernels: no workspace yet (run a registration first)");
    if (reps < 1 || !out) throw ArgFail("time_kernels: reps >= 1 and out required");
    Workspace& w = *c->last;
    const int P = w.P;
    cudaStream_t st = c->stream;
    dreg_solver_cfg s;
    dreg_solver_cfg_default(&s);
    if (scfg) {
        check_solver(scfg);
        s = *scfg;
    } else {
        s.data_term = 2;
        s.lambda = 0.1;
        s.theta = 1.0;
    }
    s.log_objective = 0;
    const bool precise = solve_precise(c->precision, s);
    if (precise) w.ensure_s64();
    const SolverParams sp = solver_params(s);
    XArgs xa = make_xargs(w, sp, false, precise);
    xa.k = 5;
    xa.coef = 0.5;
    xa.coef_prev = 0.4;
    PArgs pa = make_pargs(w, sp, false, precise);
    // the kernels a registration's solves run: the spectral-state pair when eligible
    const bool ss = solve_uses_spectral_state(w, s, xa, false, false, precise);
    const int xmode = !ss ? X_GENERAL : (ss_needs_change(s) ? X_SS : X_SSN);
    const int pmode = ss ? 2 : 0;
    if (ss) {
        pa.inv_nf = (float)(1.0 / (double)w.geo.N);
        pa.c_cur = 0.5f;
        pa.c_prev = 0.4f;
        pa.has1 = pa.has0 = 1;
        pa.U1 = reinterpret_cast<float2*>(w.BP.p);
        pa.U0 = reinterpret_cast<float2*>(w.BH.p);
        xa.ss_last = 0;
    }
    Launcher L{c};
    L(launch_state_reset(w.st.p, P, st));
    cudaEvent_t e[4];
    for (auto& ev : e) CK(cudaEventCreate(&ev));
    // warm-up
    L(launch_plane(pa, pmode, P, st));
    L(launch_xpass(xa, xmode, P, st));
    float tx = 0.f, tp = 0.f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e[0], st));
        L(launch_plane(pa, pmode, P, st));
        CK(cudaEventRecord(e[1], st));
        L(launch_xpass(xa, xmode, P, st));
        CK(cudaEventRecord(e[2], st));
        CK(cudaEventSynchronize(e[2]));
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, e[0], e[1]));
        CK(cudaEventElapsedTime(&b, e[1], e[2]));
        tp += a;
        tx += b;
    }
    for (auto& ev : e) cudaEventDestroy(ev);
    c->launches += L.count;
    const double N = (double)w.geo.N;
    const double spec = 2.0 * 3.0 * (double)w.geo.hx * (double)w.geo.lines * 8.0;  // read + write
    out[0] = tx / reps;
    out[1] = tp / reps;
    out[2] = P * (25.0 * 4.0 * N + spec);  // 16 field words read + 9 written (v, b, w), spectrum in/out
    out[3] = P * spec;
    if (ss) {
        // x-pass: grad + diff (4 words) [+ v read and written with the change norm], spectrum in/out;
        // plane: V^ in, U_{j-1} and U_{j-2} in, U_j and the filtered spectrum out = 5 half-spectra
        out[2] = P * ((xmode == X_SS ? 10.0 : 4.0) * 4.0 * N + spec);
        out[3] = P * 2.5 * spec;
    }
    out[4] = P;
    out[5] = precise ? 1.0 : 0.0;
    out[6] = ss ? (xmode == X_SS ? 1.0 : 2.0) : 0.0;
    return DREG_OK;
}

int dreg_cuda_time_kernels(dreg_cuda_ctx* c, int reps, double* out) {
    return guarded(c, [&] {
        double o[7];
        const int r = time_iteration_impl(c, nullptr, reps, o);
        for (int i = 0; i < 5; ++i) out[i] = o[i];
        return r;
    });
}

int dreg_cuda_time_iteration(dreg_cuda_ctx* c, const dreg_solver_cfg* cfg, int reps, double* out) {
    return guarded(c, [&] { return time_iteration_impl(c, cfg, reps, out); });
}

// ---- building blocks ------------------------------------------------------------
static void upload_aos(dreg_cuda_ctx* c, Workspace& w, const float* host_aos, float* dev_soa) {
    const size_t N = (size_t)w.geo.N;
    w.ensure_staging();
    CK(cudaMemcpyAsync(w.stage3.p, host_aos, sizeof(float) * 3 * N, cudaMemcpyHostToDevice, c->stream));
    CK(launch_aos_to_soa((long long)N, w.stage3.p, dev_soa, c->stream));
    c->launches += 1;
}

static void download_aos(dreg_cuda_ctx* c, Workspace& w, const float* dev_soa, float* host_aos) {
    const size_t N = (size_t)w.geo.N;
    w.ensure_staging();
    CK(launch_soa_to_aos((long long)N, dev_soa, w.stage3.p, c->stream));
    c->launches += 1;
    CK(cudaMemcpyAsync(host_aos, w.stage3.p, sizeof(float) * 3 * N, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
}

int dreg_cuda_v_update(dreg_cuda_ctx* c, const float* target, const float* warped, const float* grad,
                       const float* w_hat, const float* b_hat, dreg_dims3 d, const dreg_solver_cfg* cfg, float* out) {
    return guarded(c, [&] {
        if (!cfg) throw ArgFail("null config");
        if (cfg->data_term == 1 && !(cfg->epsilon > 0.0)) throw ArgFail("v_update_l1: epsilon must be > 0");
        check_dims(d, 1, "v_update");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.I0.p, target, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(w.I1.p, warped, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        upload_aos(c, w, grad, w.G.p);
        upload_aos(c, w, w_hat, w.WP.p);
        upload_aos(c, w, b_hat, w.BH.p);
        CK(launch_v_update(w.vg(), cfg->data_term, w.I0.p, w.I1.p, w.G.p, w.WP.p, w.BH.p, cfg->theta, cfg->epsilon,
                           w.V.p, c->stream));
        c->launches += 1;
        download_aos(c, w, w.V.p, out);
        return DREG_OK;
    });
}

int dreg_cuda_data_term_value(dreg_cuda_ctx* c, const float* target, const float* warped, const float* grad,
                              const float* v, dreg_dims3 d, int s, double* out) {
    return guarded(c, [&] {
        if (s != 1 && s != 2) throw ArgFail("data_term_value: s must be 1 or 2");
        if (!target || !warped || !grad || !v || !out) throw ArgFail("data_term_value: null buffer");
        check_dims(d, 1, "data_term_value");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.I0.p, target, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(w.I1.p, warped, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        upload_aos(c, w, grad, w.G.p);
        upload_aos(c, w, v, w.V.p);
        CK(launch_data_term(w.vg(), w.I0.p, w.I1.p, w.G.p, w.V.p, s, w.part.p, w.scal.p, w.counter.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, w.scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_trilinear_sample(dreg_cuda_ctx* c, const float* field, int ncomp, dreg_dims3 d, const double* points,
                               int64_t n, double* out) {
    return guarded(c, [&] {
        if (ncomp != 1 && ncomp != 3) throw ArgFail("trilinear_sample: ncomp must be 1 or 3");
        if (n < 0 || (n > 0 && (!field || !points || !out))) throw ArgFail("trilinear_sample: null buffer");
        check_dims(d, 1, "trilinear_sample");
        if (n == 0) return DREG_OK;
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        DevArray<double> pts, res;
        pts.alloc(3 * (size_t)n);
        res.alloc((size_t)ncomp * (size_t)n);
        CK(cudaMemcpyAsync(pts.p, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        const float* f;
        if (ncomp == 1) {
            CK(cudaMemcpyAsync(w.W0.p, field, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
            f = w.W0.p;
        } else {
            upload_aos(c, w, field, w.PHI0.p);
            f = w.PHI0.p;
        }
        CK(launch_trilinear_points(w.vg(), f, ncomp, pts.p, n, res.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, res.p, sizeof(double) * ncomp * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_w_update(dreg_cuda_ctx* c, const float* v, const float* b_hat, dreg_dims3 d, const dreg_solver_cfg* cfg,
                       float* out) {
    return guarded(c, [&] {
        if (!cfg) throw ArgFail("null config");
        if (cfg->order < 1 || cfg->order > 6) throw ArgFail("laplacian_symbol: order must be in [1, 6]");
        check_dims(d, 2, "laplacian_symbol");
        Workspace& w = c->workspace(d, 1);
        upload_aos(c, w, v, w.V.p);
        upload_aos(c, w, b_hat, w.BH.p);
        Launcher L{c};
        L(launch_state_reset(w.st.p, 1, c->stream));
        const SolverParams sp = solver_params(*cfg);
        const bool precise = c->precision == 2;  // fp64 butterflies / multiplier / storage on request
        if (precise) w.ensure_s64();
        XArgs xa = make_xargs(w, sp, false, precise);
        xa.add_bh = 1;
        L(launch_xpass(xa, X_FWD, 1, c->stream));
        PArgs pa = make_pargs(w, sp, false, precise);
        L(launch_plane(pa, 0, 1, c->stream));
        L(launch_xpass(xa, X_INV, 1, c->stream));
        c->launches += L.count;
        download_aos(c, w, w.WP.p, out);
        return DREG_OK;
    });
}

int dreg_cuda_regulariser_energy(dreg_cuda_ctx* c, const float* wfield, dreg_dims3 d, int order, double* out) {
    return guarded(c, [&] {
        if (order < 1 || order > 6) throw ArgFail("laplacian_symbol: order must be in [1, 6]");
        check_dims(d, 2, "laplacian_symbol");
        Workspace& w = c->workspace(d, 1);
        upload_aos(c, w, wfield, w.V.p);
        Launcher L{c};
        L(launch_state_reset(w.st.p, 1, c->stream));
        dreg_solver_cfg s;
        dreg_solver_cfg_default(&s);
        s.order = order;
        const SolverParams sp = solver_params(s);
        XArgs xa = make_xargs(w, sp, false);
        xa.add_bh = 0;
        L(launch_xpass(xa, X_FWD, 1, c->stream));
        PArgs pa = make_pargs(w, sp, false);
        L(launch_plane(pa, 1, 1, c->stream));
        c->launches += L.count;
        CK(cudaMemcpyAsync(out, w.energy.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_warp_image(dreg_cuda_ctx* c, const float* img, const float* disp, dreg_dims3 d, float* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "warp_image");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.I1.p, img, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        upload_aos(c, w, disp, w.PHI0.p);
        CK(launch_warp_image(w.vg(), w.I1.p, w.PHI0.p, w.W0.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, w.W0.p, sizeof(float) * N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_image_gradient(dreg_cuda_ctx* c, const float* img, dreg_dims3 d, float* out) {
    return guarded(c, [&] {
        check_dims(d, 2, "image_gradient");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.W0.p, img, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_gradient(w.vg(), w.W0.p, w.G.p, c->stream));
        c->launches += 1;
        download_aos(c, w, w.G.p, out);
        return DREG_OK;
    });
}

int dreg_cuda_compose_deformation(dreg_cuda_ctx* c, const float* disp, const float* v, dreg_dims3 d, float* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "compose_deformation");
        Workspace& w = c->workspace(d, 1);
        upload_aos(c, w, disp, w.PHI0.p);
        upload_aos(c, w, v, w.V.p);
        CK(launch_compose(w.vg(), w.PHI0.p, w.V.p, w.PHI1.p, c->stream));
        c->launches += 1;
        download_aos(c, w, w.PHI1.p, out);
        return DREG_OK;
    });
}

int dreg_cuda_jacobian(dreg_cuda_ctx* c, const float* disp, dreg_dims3 d, float* det_out, dreg_jacobian_stats* stats) {
    return guarded(c, [&] {
        check_dims(d, 3, "jacobian_determinant");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        upload_aos(c, w, disp, w.PHI0.p);
        CK(launch_jacobian(w.vg(), w.PHI0.p, w.W0.p, w.part.p, w.scal.p, w.counter.p, c->stream));
        c->launches += 1;
        double h[3];
        CK(cudaMemcpyAsync(h, w.scal.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        if (det_out) CK(cudaMemcpyAsync(det_out, w.W0.p, sizeof(float) * N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (stats) {
            stats->nonpositive = (int64_t)h[0];
            stats->interior = (int64_t)h[1];
            stats->min_det = h[2];
            stats->pct_nonpositive = 100.0 * h[0] / h[1];
        }
        return DREG_OK;
    });
}

int dreg_cuda_jacobian_device(dreg_cuda_ctx* c, const float* disp, dreg_dims3 d, float* det_out,
                              dreg_jacobian_stats* stats) {
    return guarded(c, [&] {
        check_dims(d, 3, "jacobian_determinant");
        if (!disp) throw ArgFail("null field");
        Workspace& w = c->workspace(d, 1);
        const VolGeom g{d.x, d.y, d.z, (long long)d.x * d.y * d.z};
        CK(launch_jacobian(g, disp, det_out, w.part.p, w.scal.p, w.counter.p, c->stream));
        c->launches += 1;
        double h[3];
        CK(cudaMemcpyAsync(h, w.scal.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (stats) {
            stats->nonpositive = (int64_t)h[0];
            stats->interior = (int64_t)h[1];
            stats->min_det = h[2];
            stats->pct_nonpositive = 100.0 * h[0] / h[1];
        }
        return DREG_OK;
    });
}

int dreg_cuda_normalize_intensity_pair(dreg_cuda_ctx* c, const float* a, const float* b, dreg_dims3 d, float* oa,
                                       float* ob) {
    return guarded(c, [&] {
        check_dims(d, 1, "normalize_intensity_pair");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.I0.p, a, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(w.I1.p, b, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_minmax_normalize(w.vg(), w.I0.p, w.I1.p, w.W0.p, w.W1.p, w.fscal.p, w.counter.p, c->stream));
        c->launches += 2;
        CK(cudaMemcpyAsync(oa, w.W0.p, sizeof(float) * N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(ob, w.W1.p, sizeof(float) * N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_binomial_smooth(dreg_cuda_ctx* c, const float* img, dreg_dims3 d, float* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "binomial_smooth");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.W0.p, img, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_smooth_axis(w.vg(), w.W0.p, w.W1.p, 0, 1, c->stream));
        CK(launch_smooth_axis(w.vg(), w.W1.p, w.W0.p, 1, 1, c->stream));
        CK(launch_smooth_axis(w.vg(), w.W0.p, w.W1.p, 2, 1, c->stream));
        c->launches += 3;
        CK(cudaMemcpyAsync(out, w.W1.p, sizeof(float) * N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_mean_sad(dreg_cuda_ctx* c, const float* a, const float* b, dreg_dims3 d, double* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "mean_sad");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        CK(cudaMemcpyAsync(w.W0.p, a, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(w.W1.p, b, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_sad(w.vg(), w.W0.p, w.W1.p, w.part.p, w.scal.p, w.counter.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, w.scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_downsample(dreg_cuda_ctx* c, const float* img, dreg_dims3 d, float* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "downsample");
        Workspace& w = c->workspace(d, 1);
        const size_t N = (size_t)w.geo.N;
        const VolGeom src = w.vg();
        const int ox = (d.x + 1) / 2, oy = (d.y + 1) / 2, oz = (d.z + 1) / 2;
        const VolGeom dst{ox, oy, oz, (long long)ox * oy * oz};
        CK(cudaMemcpyAsync(w.W0.p, img, sizeof(float) * N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_downsample(src, dst, w.W0.p, w.W1.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, w.W1.p, sizeof(float) * dst.N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_upsample_velocity(dreg_cuda_ctx* c, const float* v, dreg_dims3 sd, dreg_dims3 dd, float* out) {
    return guarded(c, [&] {
        check_dims(sd, 1, "upsample_velocity");
        check_dims(dd, 1, "upsample_velocity");
        if (dd.x < sd.x || dd.y < sd.y || dd.z < sd.z)
            throw ArgFail("upsample_velocity: target dims smaller than source");
        Workspace& w = c->workspace(dd, 1);  // destination-sized buffers hold both
        w.ensure_staging();
        const VolGeom src{sd.x, sd.y, sd.z, (long long)sd.x * sd.y * sd.z};
        const VolGeom dst = w.vg();
        CK(cudaMemcpyAsync(w.stage3.p, v, sizeof(float) * 3 * src.N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_aos_to_soa(src.N, w.stage3.p, w.PHI0.p, c->stream));
        CK(launch_upsample(src, dst, w.PHI0.p, w.PHI1.p, 3, c->stream));
        c->launches += 2;
        download_aos(c, w, w.PHI1.p, out);
        return DREG_OK;
    });
}

// ---- label metrics (metrics.hpp:31-42) -------------------------------------------
int dreg_cuda_warp_labels(dreg_cuda_ctx* c, const uint16_t* lbl, const float* disp, dreg_dims3 d, uint16_t* out) {
    return guarded(c, [&] {
        check_dims(d, 1, "warp_labels");
        if (!lbl || !disp || !out) throw ArgFail("warp_labels: null buffer");
        const VolGeom g{d.x, d.y, d.z, (long long)d.x * d.y * d.z};
        DevArray<uint16_t> in, res;
        DevArray<float> u;
        in.alloc((size_t)g.N);
        res.alloc((size_t)g.N);
        u.alloc(3 * (size_t)g.N);
        CK(cudaMemcpyAsync(in.p, lbl, sizeof(uint16_t) * g.N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(u.p, disp, sizeof(float) * 3 * g.N, cudaMemcpyHostToDevice, c->stream));
        CK(launch_warp_labels(g, in.p, u.p, res.p, c->stream));
        c->launches += 1;
        CK(cudaMemcpyAsync(out, res.p, sizeof(uint16_t) * g.N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return DREG_OK;
    });
}

int dreg_cuda_label_metrics(dreg_cuda_ctx* c, const uint16_t* a, const uint16_t* b, dreg_dims3 d, dreg_spacing3 sp,
                            int n_labels, const int* labels, double* dice_out, double* hd_out, int* hd_valid) {
    return guarded(c, [&] {
        check_dims(d, 1, "label metrics");
        if (!a || !b || (n_labels > 0 && !labels)) throw ArgFail("label metrics: null buffer");
        if (n_labels < 0 || n_labels > 65535) throw ArgFail("label metrics: label count out of range");
        if (!(sp.x > 0.0) || !(sp.y > 0.0) || !(sp.z > 0.0))
            throw ArgFail("label volume spacing must be positive");
        if (n_labels == 0) return DREG_OK;
        const VolGeom g{d.x, d.y, d.z, (long long)d.x * d.y * d.z};
        DevArray<uint16_t> da, db;
        DevArray<int> dl;
        da.alloc((size_t)g.N);
        db.alloc((size_t)g.N);
        dl.alloc((size_t)n_labels);
        CK(cudaMemcpyAsync(da.p, a, sizeof(uint16_t) * g.N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(db.p, b, sizeof(uint16_t) * g.N, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dl.p, labels, sizeof(int) * n_labels, cudaMemcpyHostToDevice, c->stream));
        std::vector<unsigned long long> counts(3 * (size_t)n_labels);
        std::vector<double> worst;
        DevArray<unsigned long long> dc;
        if (dice_out) {
            dc.alloc(3 * (size_t)n_labels);
            CK(launch_label_counts(g, da.p, db.p, dl.p, n_labels, dc.p, c->stream));
            c->launches += 1;
            CK(cudaMemcpyAsync(counts.data(), dc.p, sizeof(unsigned long long) * counts.size(), cudaMemcpyDeviceToHost,
                               c->stream));
        }
        DevArray<double> scratch, dw;
        DevArray<int> iscratch;
        if (hd_out || hd_valid) {
            const long long items = (long long)g.Nz * n_labels;
            // resident CTAs loop over (slice, label) items; cap the per-CTA scratch at 256 MB
            const size_t per_cta = 8 * hausdorff_scratch_doubles(g, 1) + 4 * hausdorff_scratch_ints(g, 1);
            const long long cap = std::max<long long>(1, (long long)((size_t)256 << 20) / (long long)per_cta);
            const int ctas = (int)std::min<long long>(std::min<long long>(items, 148LL * 4), cap);
            scratch.alloc(hausdorff_scratch_doubles(g, ctas));
            iscratch.alloc(hausdorff_scratch_ints(g, ctas));
            dw.alloc((size_t)items);
            worst.resize((size_t)items);
            CK(launch_hausdorff_slices(g, da.p, db.p, dl.p, n_labels, sp.x, sp.y, ctas, scratch.p, iscratch.p, dw.p,
                                       c->stream));
            c->launches += 1;
            CK(cudaMemcpyAsync(worst.data(), dw.p, sizeof(double) * items, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
        for (int j = 0; j < n_labels; ++j) {
            if (dice_out) {  // metrics.cpp:144-147
                const unsigned long long ia = counts[3 * j], ib = counts[3 * j + 1], both = counts[3 * j + 2];
                dice_out[j] = ia + ib == 0 ? 1.0 : 2.0 * (double)both / (double)(ia + ib);
            }
            if (hd_out || hd_valid) {  // metrics.cpp:172-179: slice order, fp64
                double total = 0.0;
                int contributing = 0;
                for (int z = 0; z < g.Nz; ++z) {
                    const double wz = worst[(size_t)j * g.Nz + z];
                    if (wz < 0.0) continue;
                    total += std::sqrt(wz);
                    ++contributing;
                }
                if (hd_valid) hd_valid[j] = contributing > 0;
                if (hd_out) hd_out[j] = contributing > 0 ? total / contributing : std::nan("");
            }
        }
        return DREG_OK;
    });
}

int dreg_cuda_dice(dreg_cuda_ctx* c, const uint16_t* a, const uint16_t* b, dreg_dims3 d, int label, double* out) {
    if (!out) return c ? fail(c, DREG_INVALID_ARGUMENT, "dice: null output") : DREG_INVALID_ARGUMENT;
    return dreg_cuda_label_metrics(c, a, b, d, {1.0, 1.0, 1.0}, 1, &label, out, nullptr, nullptr);
}

int dreg_cuda_hausdorff_slice_avg(dreg_cuda_ctx* c, const uint16_t* a, const uint16_t* b, dreg_dims3 d,
                                  dreg_spacing3 sp, int label, double* out) {
    if (!out) return c ? fail(c, DREG_INVALID_ARGUMENT, "hausdorff_slice_avg: null output") : DREG_INVALID_ARGUMENT;
    int valid = 0;
    const int st = dreg_cuda_label_metrics(c, a, b, d, sp, 1, &label, nullptr, out, &valid);
    if (st != DREG_OK) return st;
    if (!valid) return fail(c, DREG_INVALID_ARGUMENT, "hausdorff_slice_avg: no slice has both masks non-empty");
    return DREG_OK;
}

}  // extern "C"
