// gemm_lat.cu -- the Blackwell latency path for small fields (p < 2^16) and
// short K: ONE kernel, no encode pass, products on the 5th-generation tensor
// cores (tcgen05.mma.kind::i8, u8 x u8 -> s32 in TMEM), split-K across a
// thread-block cluster reduced through distributed shared memory, and a
// shared-memory-staged, coalesced epilogue.  The path the paper's future-work
// line asks for ("very small matrices ... a design using the finite field
// directly") and DESIGN.md §4.11.
//
// Every residue x < p < 2^16 is two unsigned bytes, x = x0 + 256 x1, so
//     sum_k a_k b_k = S0 + 256 S1 + 65536 S2,
//     S0 = A0 B0,  S1 = A0 B1 + A1 B0,  S2 = A1 B1      (byte planes),
// each S_w an exact s32 sum while 2 K 255^2 < 2^31 (K <= 16384 per CTA; the
// delayed reduction of Eq. (1), with a CTA's whole K share
// in one block), recombined exactly in 64 bits and reduced once.
//
// Work decomposition: a CTA (512 threads) owns a 128 x 64 output tile and the K
// chunks s, s + S, s + 2S, ... (128 wide) of a cluster of S CTAs (S <= 8) that
// share the tile.  Per chunk: the threads load the int32 tiles of op(A)
// (128 x 128) and op(B) (64 x 128, K-major) with coalesced loads into
// registers (the next chunk's loads are issued while the tensor core works on
// this one), reduce them mod p and write the byte planes straight into the
// 128-byte-swizzled K-major layout the UMMA descriptors read (two SMEM
// buffers); one thread issues 16 MMAs (4 byte products x 4 K steps of 32) into
// three TMEM accumulators (one per weight group w, 64 columns each).  Then each
// CTA recombines its S_w into residues mod p in shared memory, the cluster
// synchronises, and CTA s reduces its share of the tile's rows across the
// cluster through DSMEM, applies alpha / beta (C prefetched before the
// exchange) and stores whole rows (a warp writes 256 contiguous bytes).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "internal.h"
#include "modp.cuh"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int kLM = 128, kLN = 64, kLK = 128;      // tile rows, columns, K chunk (bytes of a swizzled row)
constexpr int kLThreads = 512;
constexpr int kLWarps = kLThreads / 32;
constexpr int kLMaxCluster = 8;
constexpr int kALimb = kLM * kLK;                  // 16 KB per byte plane of A
constexpr int kBLimb = kLN * kLK;                  // 8 KB per byte plane of B
constexpr int kLBuf = 2 * kALimb + 2 * kBLimb;     // one chunk's four byte planes (48 KB)
constexpr int kLSmem = 2 * kLBuf + 1024 /*align*/ + 64;
constexpr int kAItems = kLM * (kLK / 16) / kLThreads;   // 16-element items per thread: A 2, B 1
constexpr int kBItems = kLN * (kLK / 16) / kLThreads;

struct LatArgs {
    ModP M;
    unsigned long long mu64;
    const int32_t* A;
    const int32_t* B;
    int32_t* C;
    int64_t lda, ldb, ldc;
    int32_t m, n, k;
    int32_t tA, tB;
    int32_t S;          // CTAs per cluster along K
    uint32_t idesc;
    unsigned long long* trace;   // FF_TRACE=1: phase timestamps of CTA 0 (diagnostic), else null
};

__device__ __forceinline__ void lat_mark(const LatArgs& a, int i) {
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {
        unsigned long long c;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
        a.trace[i] = c;
    }
}

// Byte offset of (row r, 16-byte chunk c) in a K-major SWIZZLE_128B tile whose
// rows are 128 bytes: 8-row atoms of 1024 B, chunk index XOR-ed with r mod 8.
__device__ __forceinline__ uint32_t sw128(int r, int c) {
    return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}

// Work item `it` of a kRows x 128 K-major tile: (row, 16-byte chunk), ordered so
// that a warp's loads are coalesced along the STORED fastest dimension.
template <int kRows>
__device__ __forceinline__ void item_rc(int it, bool kmajor_src, int& r, int& c) {
    if (kmajor_src) { r = it / (kLK / 16); c = it % (kLK / 16); }   // along k within a row
    else { r = it % kRows; c = it / kRows; }                        // along r (stored row)
}

// Global loads of one item: 16 consecutive k of row r0 + r of the K-major view of
// X (kmajor_src: X[r * ld + kk], else X[kk * ld + r]); zero outside the matrix.
// Loads are unconditional, from addresses clamped into the matrix, and the
// out-of-range values are zeroed afterwards: per-element guarded loads compile
// to a branch per load (~25 instructions each), which made issuing a chunk's 48
// loads per thread instruction-bound.
__device__ __forceinline__ void load_item(const LatArgs& a, const int32_t* X, int64_t ld, bool kmajor_src, int gr,
                                          int rmax, int gk, uint32_t (&v)[16]) {
    const bool rin = gr < rmax;
    const int grc = rin ? gr : rmax - 1;
    if (kmajor_src) {
        const int32_t* src = X + static_cast<int64_t>(grc) * ld + gk;
        if (gk + 16 <= a.k && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 t4 = __ldg(reinterpret_cast<const int4*>(src) + q);
                v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
            }
        } else {
            const int32_t* row = X + static_cast<int64_t>(grc) * ld;
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = __ldg(row + min(gk + t, a.k - 1));
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (gk + t >= a.k) v[t] = 0;
        }
    } else {
        if (gk + 16 <= a.k) {
            const int32_t* src = X + static_cast<int64_t>(gk) * ld + grc;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                v[t] = __ldg(src);
                src += ld;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = __ldg(X + static_cast<int64_t>(min(gk + t, a.k - 1)) * ld + grc);
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (gk + t >= a.k) v[t] = 0;
        }
    }
    if (!rin) {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = 0;
    }
}

// Reduce 16 values mod p, split them into bytes and store one 16-byte chunk of
// each byte plane.
__device__ __forceinline__ void store_item(const LatArgs& a, const uint32_t (&v)[16], uint8_t* lo, uint8_t* hi,
                                           uint32_t off) {
    uint32_t wl[4], wh[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t x0 = residue_i32(static_cast<int32_t>(v[4 * q]), a.M);
        const uint32_t x1 = residue_i32(static_cast<int32_t>(v[4 * q + 1]), a.M);
        const uint32_t x2 = residue_i32(static_cast<int32_t>(v[4 * q + 2]), a.M);
        const uint32_t x3 = residue_i32(static_cast<int32_t>(v[4 * q + 3]), a.M);
        const uint32_t t0 = __byte_perm(x0, x1, 0x5140), t1 = __byte_perm(x2, x3, 0x5140);
        wl[q] = __byte_perm(t0, t1, 0x5410);
        wh[q] = __byte_perm(t0, t1, 0x7632);
    }
    *reinterpret_cast<uint4*>(lo + off) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    *reinterpret_cast<uint4*>(hi + off) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
}

__global__ void __launch_bounds__(kLThreads, 1) lat_gemm_kernel(const __grid_constant__ LatArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + 2 * kLBuf);   // one mbarrier per buffer
    uint32_t* holder = reinterpret_cast<uint32_t*>(done + 2);
    uint32_t* part = reinterpret_cast<uint32_t*>(smem);      // 128 x 64 residues, after the MMAs (32 KB)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int s = static_cast<int>(ptx::cluster_ctarank());   // K share of this CTA
    const int S = a.S;
    const int m0 = blockIdx.z * kLM, n0 = blockIdx.y * kLN;
    const bool akm = !a.tA, bkm = a.tB != 0;
    lat_mark(a, 0);

    if (tid == 0) {
        ptx::mbar_init(&done[0], 1);
        ptx::mbar_init(&done[1], 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc(holder, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    lat_mark(a, 1);

    const int nchunks = (a.k + kLK - 1) / kLK;
    uint32_t va[kAItems][16], vb[kBItems][16];
    auto load_chunk = [&](int ch) {
        const int k0 = ch * kLK;
#pragma unroll
        for (int i = 0; i < kAItems; ++i) {
            int r, c;
            item_rc<kLM>(tid + i * kLThreads, akm, r, c);
            load_item(a, a.A, a.lda, akm, m0 + r, a.m, k0 + 16 * c, va[i]);
        }
#pragma unroll
        for (int i = 0; i < kBItems; ++i) {
            int r, c;
            item_rc<kLN>(tid + i * kLThreads, bkm, r, c);
            load_item(a, a.B, a.ldb, bkm, n0 + r, a.n, k0 + 16 * c, vb[i]);
        }
    };
    uint32_t par[2] = {0, 0};
    int iter = 0;
    if (s < nchunks) load_chunk(s);
    lat_mark(a, 2);
    for (int ch = s; ch < nchunks; ch += S, ++iter) {
        const int buf = iter & 1;
        uint8_t* A0 = smem + buf * kLBuf;
        uint8_t* A1 = A0 + kALimb;
        uint8_t* B0 = A1 + kALimb;
        uint8_t* B1 = B0 + kBLimb;
        if (iter >= 2) {                         // the MMAs that read this buffer two chunks ago
            ptx::mbar_wait(&done[buf], par[buf]);
            par[buf] ^= 1;
        }
#pragma unroll
        for (int i = 0; i < kAItems; ++i) {
            int r, c;
            item_rc<kLM>(tid + i * kLThreads, akm, r, c);
            store_item(a, va[i], A0, A1, sw128(r, c));
        }
#pragma unroll
        for (int i = 0; i < kBItems; ++i) {
            int r, c;
            item_rc<kLN>(tid + i * kLThreads, bkm, r, c);
            store_item(a, vb[i], B0, B1, sw128(r, c));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> tensor core
        __syncthreads();
        if (iter == 0) lat_mark(a, 3);
        if (tid == 0) {
            ptx::tc_fence_after();
            const uint64_t da[2] = {ptx::smem_desc_sw128(ptx::smem_u32(A0)), ptx::smem_desc_sw128(ptx::smem_u32(A1))};
            const uint64_t db[2] = {ptx::smem_desc_sw128(ptx::smem_u32(B0)), ptx::smem_desc_sw128(ptx::smem_u32(B1))};
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t d = tmem + (i + j) * kLN;
#pragma unroll
                    for (int kk = 0; kk < kLK / kMmaK; ++kk) {
                        // the first MMA into each group's accumulator overwrites it
                        const bool over = iter == 0 && kk == 0 && !(i == 1 && j == 0);
                        ptx::mma_i8(d, da[i] + 2 * kk, db[j] + 2 * kk, a.idesc, over ? 0u : 1u);
                    }
                }
            ptx::tc_commit(&done[buf]);
        }
        if (ch + S < nchunks) load_chunk(ch + S);   // next chunk's loads overlap these MMAs
    }
    // wait for the last (up to two) chunks' MMAs
    for (int b = 0; b < 2; ++b)
        if (iter > b) ptx::mbar_wait(&done[(iter - 1 - b) & 1], par[(iter - 1 - b) & 1]);
    ptx::tc_fence_after();
    lat_mark(a, 4);

    // C rows this CTA will finish (prefetched before the cluster exchange): CTA s
    // owns rows [rA, rB) of the tile, warp w rows rA + w, rA + w + 16, ...
    const int rows_per = (kLM + S - 1) / S;
    const int rA = s * rows_per, rB = min(kLM, rA + rows_per);
    const uint32_t p = a.M.p;
    const int c2 = 2 * lane, gc = n0 + c2;            // two consecutive columns per lane
    constexpr int kMaxRows = kLM / kLWarps;           // rows per warp when S = 1
    uint32_t cin[kMaxRows][2];
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) {
        const int r = rA + warp + j * kLWarps, gr = m0 + r;
        cin[j][0] = cin[j][1] = 0;
        if (a.M.beta && r < rB && gr < a.m) {
            const int32_t* crow = a.C + static_cast<int64_t>(gr) * a.ldc;
            if (gc < a.n) cin[j][0] = static_cast<uint32_t>(crow[gc]);
            if (gc + 1 < a.n) cin[j][1] = static_cast<uint32_t>(crow[gc + 1]);
        }
    }

    // ---- recombine this CTA's weight groups: r = (S0 + 256 S1 + 65536 S2) mod p
    // warp w reads TMEM lanes 32 (w % 4) .. +31 (its rows), columns 16 (w / 4) .. +15
    {
        const int row = 32 * (warp & 3) + lane, c0 = 16 * (warp >> 2);
        const uint32_t tl = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + c0;
        uint32_t v0[16], v1[16], v2[16];
        if (iter > 0) {
            ptx::tmem_ld16(tl, v0);
            ptx::tmem_ld16(tl + kLN, v1);
            ptx::tmem_ld16(tl + 2 * kLN, v2);
            ptx::tmem_wait_ld();
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) v0[t] = v1[t] = v2[t] = 0;
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            // S_w >= 0, x < 2^46: one 64-bit Barrett reduction (fewer instructions than
            // three 32-bit residues and two Shoup products, measured)
            const unsigned long long x = static_cast<unsigned long long>(v0[t]) +
                                         (static_cast<unsigned long long>(v1[t]) << 8) +
                                         (static_cast<unsigned long long>(v2[t]) << 16);
            // column XOR (row mod 32): the 32 rows of a warp hit 32 banks (read back by rows below)
            part[row * kLN + ((c0 + t) ^ (row & 31))] = residue_u64(x, a.mu64, p);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    lat_mark(a, 5);
    if (warp == 0) ptx::tmem_dealloc(tmem, 256);
    if (S > 1) ptx::cluster_sync();   // every CTA's partial residues are in its shared memory
    else __syncthreads();
    lat_mark(a, 6);

    // ---- cluster reduction over DSMEM + alpha / beta epilogue, whole rows per warp
    const uint32_t part_s = ptx::smem_u32(part);
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) {
        const int r = rA + warp + j * kLWarps, gr = m0 + r;
        if (r >= rB || gr >= a.m) continue;
        uint32_t acc0 = 0, acc1 = 0;
        const int sc0 = c2 ^ (r & 31), sc1 = (c2 + 1) ^ (r & 31);
        if (S == 1) {
            acc0 = part[r * kLN + sc0];
            acc1 = part[r * kLN + sc1];
        } else {
            uint32_t x0[kLMaxCluster], x1[kLMaxCluster];
#pragma unroll
            for (int q = 0; q < kLMaxCluster; ++q) {      // all remote loads first, then the sums
                if (q < S) {
                    const uint32_t base = ptx::mapa(part_s, q) + static_cast<uint32_t>(r * kLN) * 4;
                    asm("ld.shared::cluster.u32 %0, [%1];" : "=r"(x0[q]) : "r"(base + sc0 * 4));
                    asm("ld.shared::cluster.u32 %0, [%1];" : "=r"(x1[q]) : "r"(base + sc1 * 4));
                }
            }
#pragma unroll
            for (int q = 0; q < kLMaxCluster; ++q)
                if (q < S) {
                    acc0 = addmod(acc0, x0[q], p);
                    acc1 = addmod(acc1, x1[q], p);
                }
        }
        int32_t* crow = a.C + static_cast<int64_t>(gr) * a.ldc;
        uint32_t o0 = mulmod_shoup(acc0, a.M.alpha, a.M.alpha_sh, p);
        uint32_t o1 = mulmod_shoup(acc1, a.M.alpha, a.M.alpha_sh, p);
        if (a.M.beta) {
            o0 = addmod(o0, mulmod_shoup(residue_i32(static_cast<int32_t>(cin[j][0]), a.M), a.M.beta, a.M.beta_sh, p), p);
            o1 = addmod(o1, mulmod_shoup(residue_i32(static_cast<int32_t>(cin[j][1]), a.M), a.M.beta, a.M.beta_sh, p), p);
        }
        if (gc + 1 < a.n && ((reinterpret_cast<uintptr_t>(crow + gc) & 7) == 0)) {
            *reinterpret_cast<int2*>(crow + gc) = make_int2(static_cast<int32_t>(o0), static_cast<int32_t>(o1));
        } else {
            if (gc < a.n) crow[gc] = static_cast<int32_t>(o0);
            if (gc + 1 < a.n) crow[gc + 1] = static_cast<int32_t>(o1);
        }
    }
    lat_mark(a, 7);
    if (S > 1) ptx::cluster_sync_relaxed();   // peers' shared memory stays valid until every CTA has read it
    lat_mark(a, 8);
}

}  // namespace

bool lat_path_ok(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    // two unsigned bytes per residue; a CTA accumulates at most k / S + 128 terms
    // per group with 2 * K * 255^2 < 2^31
    return pl.mp.p < 65536u && !pl.crt && !pl.fp64 && m > 0 && n > 0 && k > 0 && k <= 16384 &&
           m <= (int64_t{65535} * kLM) && n <= (int64_t{65535} * kLN);
}

int launch_gemm_lat(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                    const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, cudaStream_t st) {
    LatArgs a;
    a.M = pl.mp;
    a.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / pl.mp.p);
    a.A = A; a.B = B; a.C = C;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.m = static_cast<int32_t>(m); a.n = static_cast<int32_t>(n); a.k = static_cast<int32_t>(k);
    a.tA = tA ? 1 : 0; a.tB = tB ? 1 : 0;
    const int64_t tiles = ((m + kLM - 1) / kLM) * ((n + kLN - 1) / kLN);
    const int64_t nchunks = (k + kLK - 1) / kLK;
    // split K over a cluster until the grid covers the SMs (at most 8, at most the chunks)
    int S = 1;
    while (S < kLMaxCluster && S < nchunks && tiles * S * 2 <= num_sms()) S *= 2;
    if (S > nchunks) S = static_cast<int>(nchunks);
    a.S = S;
    // u8 x u8 -> s32, M = 128, N = 64, K-major operands
    a.idesc = (2u << 4) | ((static_cast<uint32_t>(kLN) >> 3) << 17) | ((static_cast<uint32_t>(kLM) >> 4) << 24);
    if (set_smem_attr(reinterpret_cast<const void*>(lat_gemm_kernel), kLSmem) != cudaSuccess) return FF_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(S), static_cast<unsigned>((n + kLN - 1) / kLN),
                       static_cast<unsigned>((m + kLM - 1) / kLM));
    cfg.blockDim = dim3(kLThreads);
    cfg.dynamicSmemBytes = kLSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(S);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    a.trace = nullptr;
    static unsigned long long* trace_buf = nullptr;
    if (knobs().trace) {   // development aid: phase timestamps of CTA 0
        if (!trace_buf) cudaMalloc(&trace_buf, 16 * sizeof(unsigned long long));
        a.trace = trace_buf;
    }
    note_launch();
    prof_gemm_begin(st);
    const cudaError_t e = cudaLaunchKernelEx(&cfg, lat_gemm_kernel, a);
    prof_gemm_end(st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_CUDA;
    }
    if (a.trace) {
        unsigned long long h[9];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[ff lat trace] m=%lld n=%lld k=%lld S=%d ns: alloc %llu load %llu store %llu mma+wait %llu "
                "recombine %llu csync %llu reduce+store %llu csync %llu\n", (long long)m, (long long)n, (long long)k, S,
                h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4], h[6] - h[5], h[7] - h[6], h[8] - h[7]);
    }
    return 0;
}

}  // namespace ff
