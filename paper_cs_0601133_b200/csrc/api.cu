#include <utility>
// api.cu -- the C ABI (include/ffgemm.h): argument checking, quick returns,
// workspace management and the launch sequence encode(A), encode(B), gemm_tc.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <set>
#include <vector>

#include "internal.h"

namespace ff {

namespace {

constexpr int kMaxDev = 64;

int g_sms[kMaxDev];
int g_arch_ok[kMaxDev];  // 0 unknown, 1 ok, 2 not sm_100

struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
};
Buf g_ws[kMaxDev];
Buf g_host_a[kMaxDev], g_host_b[kMaxDev], g_host_c[kMaxDev], g_host_ws[kMaxDev];
Buf g_scratch[kMaxDev];   // CRT residue scratch of ff_gemm_limbs
std::mutex g_mu;

// Library-owned streams for the pipelined host entry point.
struct HostStreams {
    bool init = false, ok = false;
    cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
};
HostStreams g_hs[kMaxDev];

HostStreams& host_streams(int dev) {
    HostStreams& h = g_hs[dev];
    if (!h.init) {
        h.init = true;
        h.ok = cudaStreamCreateWithFlags(&h.in, cudaStreamNonBlocking) == cudaSuccess &&
               cudaStreamCreateWithFlags(&h.comp, cudaStreamNonBlocking) == cudaSuccess &&
               cudaStreamCreateWithFlags(&h.out, cudaStreamNonBlocking) == cudaSuccess;
    }
    return h;
}

int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 || d >= kMaxDev ? 0 : d;
}

int arch_check(int dev) {
    if (dev < 0 || dev >= kMaxDev) return FF_ERR_ARCH;
    if (g_arch_ok[dev] == 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
            cudaGetLastError();
            return FF_ERR_CUDA;
        }
        g_arch_ok[dev] = (major == 10 && minor == 0) ? 1 : 2;
    }
    return g_arch_ok[dev] == 1 ? 0 : FF_ERR_ARCH;
}

int ensure(Buf& b, size_t bytes) {
    if (b.bytes >= bytes) return 0;
    if (b.ptr) {
        cudaDeviceSynchronize();
        cudaFree(b.ptr);
        b.ptr = nullptr;
        b.bytes = 0;
    }
    if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_NOMEM;
    }
    b.bytes = bytes;
    return 0;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool is_n(char t) { return t == 'N' || t == 'n'; }
bool is_t(char t) { return t == 'T' || t == 't'; }

int validate(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
             const void* B, int64_t ldb, const void* C, int64_t ldc) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (!is_n(transA) && !is_t(transA)) return -2;
    if (!is_n(transB) && !is_t(transB)) return -3;
    if (m < 0) return -4;
    if (n < 0) return -5;
    if (k < 0) return -6;
    if (!A && m > 0 && k > 0) return -8;
    const int64_t a_cols = is_n(transA) ? k : m;
    if (lda < (a_cols > 1 ? a_cols : 1)) return -9;
    if (!B && k > 0 && n > 0) return -10;
    const int64_t b_cols = is_n(transB) ? n : k;
    if (ldb < (b_cols > 1 ? b_cols : 1)) return -11;
    if (!C && m > 0 && n > 0) return -13;
    if (ldc < (n > 1 ? n : 1)) return -14;
    return 0;
}

// Measured: one level wins on c5 (L = 4, 16384^3: 18% faster),
// loses on c4 (L = 2, ~2% slower) and on c2 (4096^3, 7 short launches: 65% slower).
// So: several limbs (the MMA share of the time grows with L^2) and enough
// half-size tiles to fill the GPU a few times over.
bool winograd_auto_wins(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    const int64_t half_tiles = ((m / 2 + 255) / 256) * ((n / 2 + 255) / 256);
    return pl.info.L >= 3 && half_tiles >= 4 * (num_sms() / 2) && k >= 4096;
}

size_t ws_bytes(const Plan& pl, int64_t m, int64_t n) {
    if (pl.fp64) return f64_ws_bytes(pl, m, n, 0, 0);
    const size_t L = static_cast<size_t>(pl.info.L), kp = static_cast<size_t>(pl.info.k_pad);
    return align256(L * static_cast<size_t>(m) * kp) + align256(L * static_cast<size_t>(n) * kp) +
           align256(crt_scratch_bytes(pl));
}

int cuda_rc(cudaError_t e) { return e == cudaSuccess ? 0 : FF_ERR_CUDA; }

// One Winograd level: forced by opts->winograd == 1; auto (0)
// uses it only where it was measured to win.  Returns 1 (use), 0 (classical)
// or FF_ERR_OPTS (forced but the shape is not even).
int use_winograd(const Plan& pl, const ff_opts* opts, int64_t m, int64_t n, int64_t k) {
    const int w = opts ? opts->winograd : 0;
    if (pl.fp64) {
        // l levels of delayed Winograd (Sec. 3.2.3), only when asked for and
        // only while Corollary 3.4 allows it (the planner's exact k_winograd[l])
        if (w <= 0) return 0;
        if (k >= pl.info.k_winograd[w] && !(opts && opts->debug_unchecked_kb)) return -FF_ERR_OPTS;
        return w;
    }
    const bool even = (m % 2 == 0) && (n % 2 == 0) && (k % 2 == 0) && m >= 512 && n >= 512 && k >= 256;
    if (w == 1) return even ? 1 : -FF_ERR_OPTS;
    if (w < 0) return 0;
    return even && winograd_auto_wins(pl, m, n, k) ? 1 : 0;
}

}  // namespace

size_t gemm_ws_bytes(const Plan& pl, int64_t m, int64_t n) { return ws_bytes(pl, m, n); }

namespace {

// The whole path on device pointers.
// Small-field latency path (gemm_small.cu) for short K and small problems:
// FF_SMALL=0 never, FF_SMALL=1 whenever valid (experiments); default by size.
// The tcgen05 latency kernel (gemm_lat.cu): small_path = 2 forces it, 0 / 1 exclude it.
bool prefer_lat(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    const int mode = pl.small_mode;
    if (mode >= 0) return mode == 2;
    // measured (p = 65521, alpha = -1, beta = 1, one B200): it wins while
    // one wave of 128 x 64 tiles covers the output and each CTA has a few K chunks --
    // 512^3 18 vs 27 us (mma.sync) / 42 us (encoders + tcgen05), 256^2 x 4096 31 vs 76 us,
    // 128 x 8192 x 1024 51 vs 58 us; below K = 256 the mma.sync kernels are faster
    // (128^3: 14 vs 20 us), beyond one wave the encoder + tcgen05 path (4096^2 x 128)
    const int64_t tiles = ((m + 127) / 128) * ((n + 63) / 64);
    return k >= 256 && tiles <= num_sms() && tiles * ((k + 127) / 128) <= 1024;
}

bool prefer_small(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    const int mode = pl.small_mode;
    if (mode >= 0) return mode == 1;
    // measured (p = 65521, alpha = -1, beta = 1): 128^3 19.9 vs 31.5 us, 128 x 8192 x 128
    // 21.9 vs 33.3 us; but 512^3 40.8 vs 36.4 us, 128 x 8192 x 1024 98 vs 51 us and
    // 4096^2 x 128 233 vs 90 us -- the tcgen05 path wins beyond short K and ~2M outputs
    return k <= 256 && m * n <= (int64_t{1} << 21);
}

// The cp.async variant for canonical operands (internal callers): FF_SMALL as above.
bool prefer_small_canon(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    const int mode = pl.small_mode;
    if (mode >= 0) return mode == 1;
    // measured against the tcgen05 path (p = 65521, alpha = -1, beta = 1): 512^3 21 vs
    // 36 us, 128 x 8192 x 128 20 vs 33 us, 128 x 8192 x 1024 51 vs 51 us, 1024^3
    // 51 vs 41 us, 4096^2 x 128 146 vs 90 us
    return k <= 1024 && m * n <= (int64_t{1} << 21) && m * n * k < (int64_t{1} << 30);
}

// The same for 2^16 <= p < 2^31 (3-4 bytes per residue): FF_SMALL as above.
bool prefer_small_wide(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    const int mode = pl.small_mode;
    if (mode >= 0) return mode == 1;
    return k <= 1024 && m * n <= (int64_t{1} << 21) && m * n * k < (int64_t{1} << 29);
}

int run(const Plan& pl, char transA, char transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
        int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st) {
    if (k == 0 || pl.mp.alpha == 0) return cuda_rc(launch_scale_c(pl.mp, m, n, C, ldc, st));
    if (pl.fp64) return run_f64(pl, 0, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb, C, ldc, ws, st);
    // The small paths read A and B while other CTAs write C, so C must not overlap
    // them (an in-place product, e.g. LQUP's U_rest = L11^-1 A_rest, takes the
    // tcgen05 path, which reads only the encoded planes).  Conservative span test.
    auto span = [](const int32_t* X, int64_t rows, int64_t cols, int64_t ld) {
        const uintptr_t lo = reinterpret_cast<uintptr_t>(X);
        return std::make_pair(lo, lo + static_cast<uintptr_t>(((rows - 1) * ld + cols) * 4));
    };
    const auto sa = is_t(transA) ? span(A, k, m, lda) : span(A, m, k, lda);
    const auto sb = is_t(transB) ? span(B, n, k, ldb) : span(B, k, n, ldb);
    const auto sc = span(C, m, n, ldc);
    const bool c_disjoint = (sc.second <= sa.first || sa.second <= sc.first) &&
                            (sc.second <= sb.first || sb.second <= sc.first);
    // the tcgen05 latency kernel: one launch, no encoders (C must not overlap A, B)
    if (pl.all_auto && c_disjoint && lat_path_ok(pl, m, n, k) && prefer_lat(pl, m, n, k))
        return launch_gemm_lat(pl, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb, C, ldc, st);
    // (the canonical-input variants handle overlap with a grid barrier instead)
    if (pl.all_auto && small_canon_ok(pl, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb) &&
        prefer_small_canon(pl, m, n, k)) {
        const int e = launch_gemm_small_canon(pl, m, n, k, A, lda, B, ldb, C, ldc, !c_disjoint, st);
        if (e != FF_ERR_INTERNAL) return e;
    } else if (pl.all_auto && small_stream_ok(pl, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb) &&
               prefer_small_canon(pl, m, n, k)) {
        // raw inputs, not transposed: the same streaming kernel reduces each slice in shared memory
        const int e = launch_gemm_small_canon(pl, m, n, k, A, lda, B, ldb, C, ldc, !c_disjoint, st, true);
        if (e != FF_ERR_INTERNAL) return e;
    } else if (pl.all_auto && small_wide_ok(pl, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb) &&
               prefer_small_wide(pl, m, n, k)) {
        const int e = launch_gemm_small_wide(pl, m, n, k, A, lda, B, ldb, C, ldc, !c_disjoint, st);
        if (e != FF_ERR_INTERNAL) return e;
    }
    if (pl.all_auto && c_disjoint && small_path_ok(pl, m, n, k) && prefer_small(pl, m, n, k))
        return launch_gemm_small(pl, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb, C, ldc, st);
    int8_t* al = static_cast<int8_t*>(ws);
    int8_t* bl = al + align256(static_cast<size_t>(pl.info.L) * m * pl.info.k_pad);
    int8_t* scratch = bl + align256(static_cast<size_t>(pl.info.L) * n * pl.info.k_pad);
    int e = cuda_rc(launch_encode(pl, is_n(transA) ? 1 : 0, m, k, A, lda, al, st));
    if (e) return e;
    e = cuda_rc(launch_encode(pl, is_t(transB) ? 1 : 0, n, k, B, ldb, bl, st));
    if (e) return e;
    return launch_gemm_tc(pl, m, n, k, al, bl, C, ldc, scratch, st);
}

}  // namespace

int gemm_dev(const Plan& pl, char transA, char transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
             int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st) {
    return run(pl, transA, transB, m, n, k, A, lda, B, ldb, C, ldc, ws, st);
}

int check_device() { return arch_check(cur_dev()); }

cudaError_t set_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    const int dev = cur_dev();
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({dev, fn})) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({dev, fn});
    return e;
}

namespace {
struct Prof {
    std::mutex mu;
    std::atomic<bool> on{false};
    std::atomic<long long> launches{0};
    int dev = -1;
    std::vector<cudaEvent_t> ev;   // 2 per GEMM launch
    int used = 0, cap = 0;
};
Prof g_prof;
}  // namespace

void note_launch(int n) {
    if (g_prof.on.load(std::memory_order_relaxed)) g_prof.launches.fetch_add(n, std::memory_order_relaxed);
}

void prof_gemm_begin(cudaStream_t st) {
    if (!g_prof.on.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (g_prof.used >= g_prof.cap || cur_dev() != g_prof.dev) return;
    cudaEventRecord(g_prof.ev[2 * g_prof.used], st);
}

void prof_gemm_end(cudaStream_t st) {
    if (!g_prof.on.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (g_prof.used >= g_prof.cap || cur_dev() != g_prof.dev) return;
    cudaEventRecord(g_prof.ev[2 * g_prof.used + 1], st);
    ++g_prof.used;
}

namespace {
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
}  // namespace

const Knobs& knobs() {
    static const Knobs k = [] {
        Knobs v;
        v.small = env_int("FF_SMALL", -1);
        v.pdl = getenv("FF_NOPDL") == nullptr;
        v.trace = getenv("FF_TRACE") != nullptr;
        v.raster = env_int("FF_RASTER", 0);
        v.hints = env_int("FF_HINTS", -1);
        v.korder = env_int("FF_KORDER", 0);
        v.kbloc = getenv("FF_KBLOC") ? atoll(getenv("FF_KBLOC")) : 0;
        v.enc_notma = getenv("FF_ENC_NOTMA") != nullptr;
        v.wide = getenv("FF_NOWIDE") == nullptr;
        v.wdelta = env_int("FF_WDELTA", 0);
        v.wdelta_wb = env_int("FF_WDELTA_WB", 0);
#ifdef FF_EXPERIMENTS
        v.throttle = env_int("FF_THROTTLE", 0);
        v.die_aware = getenv("FF_DIE_AWARE") != nullptr && getenv("FF_NO_DIE_AWARE") == nullptr;
#else
        v.throttle = 0;
        v.die_aware = false;
#endif
        return v;
    }();
    return k;
}

int num_sms() {
    const int d = cur_dev();
    if (g_sms[d] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        g_sms[d] = v;
    }
    return g_sms[d];
}

}  // namespace ff

using namespace ff;

extern "C" {

int ff_version(void) { return 100; }

const char* ff_strerror(int code) {
    switch (code) {
        case FF_OK: return "success";
        case FF_ERR_CUDA: return "CUDA runtime/driver error";
        case FF_ERR_NOMEM: return "out of device memory or workspace too small";
        case FF_ERR_ARCH: return "device is not an sm_100 (B200) GPU";
        case FF_ERR_OPTS: return "invalid ff_opts";
        case FF_ERR_INTERNAL: return "internal planner error";
        default: break;
    }
    if (code < 0) {
        switch (-code) {
            case 1: return "invalid argument 1 (p)";
            case 2: return "invalid argument 2 (transA)";
            case 3: return "invalid argument 3 (transB)";
            case 4: return "invalid argument 4 (m)";
            case 5: return "invalid argument 5 (n)";
            case 6: return "invalid argument 6 (k)";
            case 8: return "invalid argument 8 (A)";
            case 9: return "invalid argument 9 (lda)";
            case 10: return "invalid argument 10 (B)";
            case 11: return "invalid argument 11 (ldb)";
            case 13: return "invalid argument 13 (C)";
            case 14: return "invalid argument 14 (ldc)";
            case 16: return "invalid argument 16 (workspace)";
            default: return "invalid argument";
        }
    }
    return "unknown error";
}

int ff_device_check(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_CUDA;
    }
    if (device < 0 || device >= n) return FF_ERR_ARCH;
    return arch_check(device);
}

int ff_plan_query(uint32_t p, int64_t k, const ff_opts* opts, ff_plan_info* out) {
    if (!out) return -4;
    Plan pl;
    int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    *out = pl.info;
    return 0;
}

size_t ff_gemm_workspace_size(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
                              const ff_opts* opts) {
    (void)transA;
    (void)transB;
    if (m < 0 || n < 0 || k < 0) return 0;
    Plan pl;
    if (make_plan(p, k, opts, &pl)) return 0;
    size_t need = ws_bytes(pl, m, n);
    if (pl.fp64) {
        const int lv = use_winograd(pl, opts, m, n, k);
        return f64_ws_bytes(pl, m, n, k, lv > 0 ? lv : 0);
    }
    if (use_winograd(pl, opts, m, n, k) == 1) {
        Plan half;
        if (make_plan(p, k / 2, opts, &half)) return 0;
        need = std::max(need, winograd_ws_bytes(half, m, n, k));
    }
    return need;
}

int ff_gemm_winograd_levels(uint32_t p, int64_t m, int64_t n, int64_t k, const ff_opts* opts, int32_t* levels) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    if (k < 0) return -4;
    if (!levels) return -6;
    Plan pl;
    const int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    *levels = 0;
    if (m == 0 || n == 0 || k == 0) return 0;
    const int w = use_winograd(pl, opts, m, n, k);
    if (w < 0) return -w;
    *levels = w;
    return 0;
}

int ff_gemm_ex(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k, uint32_t alpha,
               const int32_t* A, int64_t lda, const int32_t* B, int64_t ldb, uint32_t beta, int32_t* C,
               int64_t ldc, const ff_opts* opts, void* workspace, size_t workspace_bytes, void* stream) {
    int e = validate(p, transA, transB, m, n, k, A, lda, B, ldb, C, ldc);
    if (e) return e;
    if (m == 0 || n == 0) return 0;
    Plan pl;
    e = make_plan(p, k, opts, &pl);
    if (e) return e;
    set_scalars(&pl, alpha, beta);
    const int wino = (k == 0 || pl.mp.alpha == 0) ? 0 : use_winograd(pl, opts, m, n, k);
    if (wino < 0) return -wino;
    Plan half;
    if (wino && !pl.fp64) {
        if ((e = make_plan(p, k / 2, opts, &half))) return e;
        set_scalars(&half, alpha, beta);
    }
    const int dev = cur_dev();
    e = arch_check(dev);
    if (e) return e;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t need = pl.fp64 ? f64_ws_bytes(pl, m, n, k, wino)
                                : wino ? winograd_ws_bytes(half, m, n, k) : ws_bytes(pl, m, n);
    auto go = [&](void* w) {
        if (pl.fp64 && wino)
            return run_f64(pl, wino, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb, C, ldc, w, st);
        return wino ? run_winograd(half, is_t(transA), is_t(transB), m, n, k, A, lda, B, ldb, C, ldc, w, st)
                    : run(pl, transA, transB, m, n, k, A, lda, B, ldb, C, ldc, w, st);
    };
    if (workspace) {
        if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255)) return -16;
        return go(workspace);
    }
    std::lock_guard<std::mutex> lk(g_mu);
    e = ensure(g_ws[dev], need);
    if (e) return e;
    return go(g_ws[dev].ptr);
}

int ff_gemm(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k, uint32_t alpha,
            const int32_t* A, int64_t lda, const int32_t* B, int64_t ldb, uint32_t beta, int32_t* C, int64_t ldc) {
    return ff_gemm_ex(p, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, nullptr, nullptr, 0,
                      nullptr);
}

int ff_gemm_host(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k, uint32_t alpha,
                 const int32_t* A, int64_t lda, const int32_t* B, int64_t ldb, uint32_t beta, int32_t* C,
                 int64_t ldc, const ff_opts* opts) {
    int e = validate(p, transA, transB, m, n, k, A, lda, B, ldb, C, ldc);
    if (e) return e;
    if (m == 0 || n == 0) return 0;
    Plan pl;
    e = make_plan(p, k, opts, &pl);
    if (e) return e;
    if (pl.fp64) return FF_ERR_OPTS;                 // the fp64 engine has no host pipeline
    if (opts && opts->host_block < 0) return FF_ERR_OPTS;
    set_scalars(&pl, alpha, beta);
    const int dev = cur_dev();
    e = arch_check(dev);
    if (e) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    HostStreams& hs = host_streams(dev);
    if (!hs.ok) return FF_ERR_CUDA;
    const bool tA = is_t(transA), tB = is_t(transB);
    const bool beta_nz = pl.mp.beta != 0;
    const int64_t ar = tA ? k : m, ac = tA ? m : k;   // stored A (dense copy on device)
    const int64_t br = tB ? n : k, bc = tB ? k : n;   // stored B
    if ((e = ensure(g_host_c[dev], sizeof(int32_t) * (size_t)(m * n)))) return e;
    int32_t* dC = static_cast<int32_t*>(g_host_c[dev].ptr);
    if (k == 0 || pl.mp.alpha == 0) {             // C <- beta C
        if (beta_nz && cudaMemcpy2DAsync(dC, n * 4, C, ldc * 4, n * 4, m, cudaMemcpyHostToDevice, hs.comp))
            return FF_ERR_CUDA;
        if ((e = cuda_rc(launch_scale_c(pl.mp, m, n, dC, n, hs.comp)))) return e;
        if (cudaMemcpy2DAsync(C, ldc * 4, dC, n * 4, n * 4, m, cudaMemcpyDeviceToHost, hs.comp)) return FF_ERR_CUDA;
        return cudaStreamSynchronize(hs.comp) == cudaSuccess ? 0 : FF_ERR_CUDA;
    }
    // Blocks of C: P row panels x Q column chunks, multiples of 256.
    int64_t hb = (opts && opts->host_block > 0) ? opts->host_block : 4096;
    hb = (hb + 255) / 256 * 256;
    const int64_t P = (m + hb - 1) / hb, Q = (n + hb - 1) / hb;
    const int64_t mb = std::min<int64_t>(hb, m), nb = std::min<int64_t>(hb, n);
    const size_t L = static_cast<size_t>(pl.info.L), kp = static_cast<size_t>(pl.info.k_pad);
    const size_t a_panel = align256(L * mb * kp), b_chunk = align256(L * nb * kp);
    if ((e = ensure(g_host_a[dev], sizeof(int32_t) * (size_t)(ar * ac)))) return e;
    if ((e = ensure(g_host_b[dev], sizeof(int32_t) * (size_t)(br * bc)))) return e;
    const size_t scr = align256(crt_scratch_bytes(pl));
    if ((e = ensure(g_host_ws[dev], a_panel * P + b_chunk * Q + scr))) return e;
    int32_t* dA = static_cast<int32_t*>(g_host_a[dev].ptr);
    int32_t* dB = static_cast<int32_t*>(g_host_b[dev].ptr);
    int8_t* wsA = static_cast<int8_t*>(g_host_ws[dev].ptr);
    int8_t* wsB = wsA + a_panel * P;
    int8_t* scratch = wsB + b_chunk * Q;    // GEMMs of the blocks run in order on hs.comp
    std::vector<cudaEvent_t> evs;
    auto mkev = [&]() {
        cudaEvent_t ev = nullptr;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        evs.push_back(ev);
        return ev;
    };
    std::vector<cudaEvent_t> evA(P), evB(Q), evCin(P * Q), evG(P * Q);
    for (auto& x : evA) x = mkev();
    for (auto& x : evB) x = mkev();
    for (auto& x : evG) x = mkev();
    if (beta_nz)
        for (auto& x : evCin) x = mkev();
    auto rows_of = [&](int64_t i, int64_t& r0, int64_t& r1) { r0 = i * hb; r1 = std::min(m, r0 + hb); };
    auto cols_of = [&](int64_t j, int64_t& c0, int64_t& c1) { c0 = j * hb; c1 = std::min(n, c0 + hb); };
    bool fail = false;
    auto chk = [&](cudaError_t x) { if (x != cudaSuccess) fail = true; };
    // Block order: "growing squares" s = 0, 1, ...: after row panel s of A and
    // column chunk s of B have arrived, the new blocks (s, 0..s) and (0..s-1, s)
    // are computable.  Copies in, GEMMs and copies out all follow this order, so
    // the device->host stream (the PCIe floor: all of C) starts after the first
    // panel + chunk and is never starved afterwards.
    std::vector<std::pair<int64_t, int64_t>> order;
    const int64_t S = std::max(P, Q);
    for (int64_t sq = 0; sq < S; ++sq) {
        if (sq < P)
            for (int64_t j = 0; j <= std::min(sq, Q - 1); ++j) order.push_back({sq, j});
        if (sq < Q)
            for (int64_t i = 0; i < std::min(sq, P); ++i) order.push_back({i, sq});
    }
    // ---- host -> device (stream hs.in)
    for (int64_t sq = 0; sq < S && !fail; ++sq) {
        if (sq < P) {
            int64_t r0, r1;
            rows_of(sq, r0, r1);
            const int64_t rows = r1 - r0;
            if (!tA) chk(cudaMemcpy2DAsync(dA + r0 * k, k * 4, A + r0 * lda, lda * 4, k * 4, rows, cudaMemcpyHostToDevice, hs.in));
            else chk(cudaMemcpy2DAsync(dA + r0, m * 4, A + r0, lda * 4, rows * 4, k, cudaMemcpyHostToDevice, hs.in));
            chk(cudaEventRecord(evA[sq], hs.in));
        }
        if (sq < Q) {
            int64_t c0, c1;
            cols_of(sq, c0, c1);
            const int64_t cols = c1 - c0;
            if (!tB) chk(cudaMemcpy2DAsync(dB + c0, n * 4, B + c0, ldb * 4, cols * 4, k, cudaMemcpyHostToDevice, hs.in));
            else chk(cudaMemcpy2DAsync(dB + c0 * k, k * 4, B + c0 * ldb, ldb * 4, k * 4, cols, cudaMemcpyHostToDevice, hs.in));
            chk(cudaEventRecord(evB[sq], hs.in));
        }
        if (beta_nz)
            for (const auto& blk : order) {
                if (std::max(blk.first, blk.second) != sq) continue;
                int64_t r0, r1, c0, c1;
                rows_of(blk.first, r0, r1);
                cols_of(blk.second, c0, c1);
                chk(cudaMemcpy2DAsync(dC + r0 * n + c0, n * 4, C + r0 * ldc + c0, ldc * 4, (c1 - c0) * 4, r1 - r0,
                                      cudaMemcpyHostToDevice, hs.in));
                chk(cudaEventRecord(evCin[blk.first * Q + blk.second], hs.in));
            }
    }
    // ---- compute (stream hs.comp): encode each operand block once, GEMM each C block
    std::vector<char> encA(P, 0), encB(Q, 0);
    for (const auto& blk : order) {
        if (fail) break;
        const int64_t i = blk.first, j = blk.second;
        int64_t r0, r1, c0, c1;
        rows_of(i, r0, r1);
        cols_of(j, c0, c1);
        int8_t* Al = wsA + a_panel * i;
        int8_t* Bl = wsB + b_chunk * j;
        if (!encA[i]) {
            chk(cudaStreamWaitEvent(hs.comp, evA[i], 0));
            chk(launch_encode(pl, tA ? 0 : 1, r1 - r0, k, tA ? dA + r0 : dA + r0 * k, tA ? m : k, Al, hs.comp));
            encA[i] = 1;
        }
        if (!encB[j]) {
            chk(cudaStreamWaitEvent(hs.comp, evB[j], 0));
            chk(launch_encode(pl, tB ? 1 : 0, c1 - c0, k, tB ? dB + c0 * k : dB + c0, tB ? k : n, Bl, hs.comp));
            encB[j] = 1;
        }
        if (beta_nz) chk(cudaStreamWaitEvent(hs.comp, evCin[i * Q + j], 0));
        if (launch_gemm_tc(pl, r1 - r0, c1 - c0, k, Al, Bl, dC + r0 * n + c0, n, scratch, hs.comp)) fail = true;
        chk(cudaEventRecord(evG[i * Q + j], hs.comp));
    }
    // ---- device -> host (stream hs.out): each C block as soon as its GEMM is done
    for (const auto& blk : order) {
        if (fail) break;
        int64_t r0, r1, c0, c1;
        rows_of(blk.first, r0, r1);
        cols_of(blk.second, c0, c1);
        chk(cudaStreamWaitEvent(hs.out, evG[blk.first * Q + blk.second], 0));
        chk(cudaMemcpy2DAsync(C + r0 * ldc + c0, ldc * 4, dC + r0 * n + c0, n * 4, (c1 - c0) * 4, r1 - r0,
                              cudaMemcpyDeviceToHost, hs.out));
    }
    const cudaError_t s1 = cudaStreamSynchronize(hs.in);
    const cudaError_t s2 = cudaStreamSynchronize(hs.comp);
    const cudaError_t s3 = cudaStreamSynchronize(hs.out);
    for (auto ev : evs) cudaEventDestroy(ev);
    return (fail || s1 || s2 || s3) ? FF_ERR_CUDA : 0;
}

int ff_encode(uint32_t p, int64_t k, const ff_opts* opts, int kmajor_src, int64_t rows, const int32_t* X,
              int64_t ldx, int8_t* limbs, void* stream) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (k < 0) return -2;
    if (rows < 0) return -4;
    if (!X && rows > 0 && k > 0) return -5;
    if (ldx < 1 || (kmajor_src && ldx < k) || (!kmajor_src && ldx < rows)) return -6;
    if ((!limbs && rows > 0 && k > 0) || (reinterpret_cast<uintptr_t>(limbs) & 15)) return -7;
    Plan pl;
    int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    if (pl.fp64) return FF_ERR_OPTS;                 // int8 planes only
    e = arch_check(cur_dev());
    if (e) return e;
    return cuda_rc(launch_encode(pl, kmajor_src, rows, k, X, ldx, limbs, static_cast<cudaStream_t>(stream)));
}

int ff_gemm_limbs(uint32_t p, int64_t m, int64_t n, int64_t k, const ff_opts* opts, uint32_t alpha,
                  const int8_t* A_limbs, const int8_t* B_limbs, uint32_t beta, int32_t* C, int64_t ldc,
                  void* stream) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    if (k < 0) return -4;
    if (m == 0 || n == 0) return 0;
    if (k > 0 && (!A_limbs || (reinterpret_cast<uintptr_t>(A_limbs) & 15))) return -7;
    if (k > 0 && (!B_limbs || (reinterpret_cast<uintptr_t>(B_limbs) & 15))) return -8;
    if (!C) return -10;
    if (ldc < (n > 1 ? n : 1)) return -11;
    Plan pl;
    int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    if (pl.fp64) return FF_ERR_OPTS;                 // int8 planes only
    set_scalars(&pl, alpha, beta);
    e = arch_check(cur_dev());
    if (e) return e;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (k == 0 || pl.mp.alpha == 0) return cuda_rc(launch_scale_c(pl.mp, m, n, C, ldc, st));
    void* scratch = nullptr;
    if (const size_t sb = crt_scratch_bytes(pl)) {
        std::lock_guard<std::mutex> lk(g_mu);
        const int dev = cur_dev();
        if ((e = ensure(g_scratch[dev], sb))) return e;
        scratch = g_scratch[dev].ptr;
    }
    return launch_gemm_tc(pl, m, n, k, A_limbs, B_limbs, C, ldc, scratch, st);
}

int ff_fill_uniform(int32_t* X, int64_t rows, int64_t cols, int64_t ld, uint32_t p, uint64_t seed,
                    uint32_t stream_id, int64_t index0, void* stream) {
    if (rows < 0) return -2;
    if (cols < 0) return -3;
    if (ld < (cols > 1 ? cols : 1)) return -4;
    if (p < 2 || p >= (1u << 31)) return -5;
    if (!X && rows * cols > 0) return -1;
    int e = arch_check(cur_dev());
    if (e) return e;
    return cuda_rc(launch_fill_uniform(X, rows, cols, ld, p, seed, stream_id, index0,
                                       static_cast<cudaStream_t>(stream)));
}

int ff_prof_start(int32_t capacity) {
    if (capacity < 0 || capacity > (1 << 20)) return -1;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    const int dev = cur_dev();
    if (g_prof.dev != dev) {
        for (cudaEvent_t e : g_prof.ev) cudaEventDestroy(e);
        g_prof.ev.clear();
        g_prof.dev = dev;
    }
    while (static_cast<int>(g_prof.ev.size()) < 2 * capacity) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return FF_ERR_CUDA;
        g_prof.ev.push_back(e);
    }
    g_prof.cap = capacity;
    g_prof.used = 0;
    g_prof.launches.store(0);
    g_prof.on.store(true);
    return 0;
}

int ff_prof_stop(float* gemm_ms, int32_t cap, int64_t* launches) {
    g_prof.on.store(false);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (launches) *launches = g_prof.launches.load();
    const int n = g_prof.used;
    for (int i = 0; i < n && i < cap && gemm_ms; ++i) {
        if (cudaEventSynchronize(g_prof.ev[2 * i + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&gemm_ms[i], g_prof.ev[2 * i], g_prof.ev[2 * i + 1]) != cudaSuccess)
            return -FF_ERR_CUDA;
    }
    g_prof.used = 0;
    return n;
}

}  // extern "C"
