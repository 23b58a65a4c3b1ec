// winograd.cu -- one level of Winograd's variant of Strassen (§3.2,
// l.235-276), fused with the tcgen05 limb GEMM.
//
// Table 2 (l.263-276) schedules C <- alpha A B + beta C with 7 half-size
// products; step 16 prints "A12 T4", which must be A22 (App. A.2, l.935;
// DESIGN.md reading R9).  In the paper the pre-additions S1..S4, T1..T4 are
// left unreduced (Thm 3.1 bounds their growth); here they are reduced mod p
// (and later re-centred by the encoder), so the limb count and the k-block
// bound of the half-size products are those of plain inputs.
//
//   S1 = A21 + A22   S2 = S1 - A11   S3 = A11 - A21   S4 = A12 - S2
//   T1 = B12 - B11   T2 = B22 - T1   T3 = B22 - B12   T4 = T2 - B21
//   P1 = A11 B11  P2 = A12 B21  P3 = S4 B22  P4 = A22 T4  P5 = S1 T1  P6 = S2 T2  P7 = S3 T3
//   C11 = a(P1 + P2)            + b C11
//   C12 = a(P1 + P6 + P5 + P3)  + b C12
//   C21 = a(P1 + P6 + P7 - P4)  + b C21
//   C22 = a(P1 + P6 + P7 + P5)  + b C22
//
// Instead of Table 2's temporaries X1..X3 and post-additions, each product's
// fused epilogue adds +-alpha P_i (mod p) directly into every C quadrant it
// contributes to, so the products are never stored -- except two temporaries
// (T = P1 and U = P6 + T) that later epilogues add, which keep every product at
// <= 2 read-modify-written quadrants (schedule in run_winograd).
#include <cuda_runtime.h>

#include <vector>

#include "internal.h"
#include "modp.cuh"

namespace ff {

namespace {

__device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, uint32_t p) {
    return a >= b ? a - b : a + (p - b);
}

// Stored-orientation quadrant sums (elementwise, so transposed storage just
// transposes every operand consistently).  which = 0: A side (S1..S4 from
// q11, q12, q21, q22), which = 1: B side (T1..T4).
__global__ void __launch_bounds__(256) preadd_kernel(ModP M, int which, int64_t rows, int64_t cols,
                                                     const int32_t* __restrict__ q11, const int32_t* __restrict__ q12,
                                                     const int32_t* __restrict__ q21, const int32_t* __restrict__ q22,
                                                     int64_t ld, int32_t* __restrict__ o1, int32_t* __restrict__ o2,
                                                     int32_t* __restrict__ o3, int32_t* __restrict__ o4) {
    auto sums = [&](int32_t a11, int32_t a12, int32_t a21, int32_t a22, uint32_t (&s)[4]) {
        const uint32_t x11 = residue_i32(a11, M), x12 = residue_i32(a12, M);
        const uint32_t x21 = residue_i32(a21, M), x22 = residue_i32(a22, M);
        if (which == 0) {
            s[0] = addmod(x21, x22, M.p);      // S1 = A21 + A22
            s[1] = submod(s[0], x11, M.p);     // S2 = S1 - A11
            s[2] = submod(x11, x21, M.p);      // S3 = A11 - A21
            s[3] = submod(x12, s[1], M.p);     // S4 = A12 - S2
        } else {
            s[0] = submod(x12, x11, M.p);      // T1 = B12 - B11
            s[1] = submod(x22, s[0], M.p);     // T2 = B22 - T1
            s[2] = submod(x22, x12, M.p);      // T3 = B22 - B12
            s[3] = submod(s[1], x21, M.p);     // T4 = T2 - B21
        }
    };
    // 16-byte accesses (4 elements per thread) when every row of every operand is
    // 16-byte aligned: the kernel is HBM-bound (4 x 4 B read + 4 x 4 B written per element)
    const bool vec = (ld % 4 == 0) && (cols % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(q11) | reinterpret_cast<uintptr_t>(q12) |
                       reinterpret_cast<uintptr_t>(q21) | reinterpret_cast<uintptr_t>(q22) |
                       reinterpret_cast<uintptr_t>(o1) | reinterpret_cast<uintptr_t>(o2) |
                       reinterpret_cast<uintptr_t>(o3) | reinterpret_cast<uintptr_t>(o4)) & 15) == 0;
    if (vec) {
        for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
            for (int64_t c = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); c < cols;
                 c += 4 * (int64_t)gridDim.x * blockDim.x) {
                const int64_t i = r * ld + c, o = r * cols + c;
                const int4 v11 = __ldg(reinterpret_cast<const int4*>(q11 + i));
                const int4 v12 = __ldg(reinterpret_cast<const int4*>(q12 + i));
                const int4 v21 = __ldg(reinterpret_cast<const int4*>(q21 + i));
                const int4 v22 = __ldg(reinterpret_cast<const int4*>(q22 + i));
                uint32_t s0[4], s1[4], s2[4], s3[4];
                sums(v11.x, v12.x, v21.x, v22.x, s0);
                sums(v11.y, v12.y, v21.y, v22.y, s1);
                sums(v11.z, v12.z, v21.z, v22.z, s2);
                sums(v11.w, v12.w, v21.w, v22.w, s3);
                *reinterpret_cast<int4*>(o1 + o) = make_int4(s0[0], s1[0], s2[0], s3[0]);
                *reinterpret_cast<int4*>(o2 + o) = make_int4(s0[1], s1[1], s2[1], s3[1]);
                *reinterpret_cast<int4*>(o3 + o) = make_int4(s0[2], s1[2], s2[2], s3[2]);
                *reinterpret_cast<int4*>(o4 + o) = make_int4(s0[3], s1[3], s2[3], s3[3]);
            }
        }
        return;
    }
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = r * ld + c, o = r * cols + c;
            uint32_t s[4];
            sums(__ldg(q11 + i), __ldg(q12 + i), __ldg(q21 + i), __ldg(q22 + i), s);
            o1[o] = static_cast<int32_t>(s[0]);
            o2[o] = static_cast<int32_t>(s[1]);
            o3[o] = static_cast<int32_t>(s[2]);
            o4[o] = static_cast<int32_t>(s[3]);
        }
    }
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Pointer to quadrant (r, c) of op(X) inside the stored X (ld), with op(X) halves hr x hc.
const int32_t* quad(const int32_t* X, int64_t ld, bool trans, int64_t hr, int64_t hc, int r, int c) {
    return trans ? X + c * hc * ld + r * hr : X + r * hr * ld + c * hc;
}

}  // namespace

size_t winograd_ws_bytes(const Plan& half, int64_t m, int64_t n, int64_t k) {
    const size_t hm = m / 2, hn = n / 2, hk = k / 2;
    const size_t L = half.info.L, kp = half.info.k_pad;
    return 4 * align256(4 * hm * hk) + 4 * align256(4 * hk * hn) + 7 * align256(L * hm * kp) +
           7 * align256(L * hn * kp) + align256(crt_scratch_bytes(half)) + 2 * align256(4 * hm * hn);
}

int run_winograd(const Plan& half, bool transA, bool transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
                 int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st) {
    const int64_t hm = m / 2, hn = n / 2, hk = k / 2;
    const size_t L = half.info.L, kp = half.info.k_pad;
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto take = [&](size_t bytes) { uint8_t* p = w; w += align256(bytes); return p; };
    int32_t* S[4];
    int32_t* T[4];
    for (int i = 0; i < 4; ++i) S[i] = reinterpret_cast<int32_t*>(take(4 * hm * hk));
    for (int i = 0; i < 4; ++i) T[i] = reinterpret_cast<int32_t*>(take(4 * hk * hn));
    int8_t* Al[7];
    int8_t* Bl[7];
    for (int i = 0; i < 7; ++i) Al[i] = reinterpret_cast<int8_t*>(take(L * hm * kp));
    for (int i = 0; i < 7; ++i) Bl[i] = reinterpret_cast<int8_t*>(take(L * hn * kp));
    void* scratch = take(crt_scratch_bytes(half));   // CRT residue scratch, shared by the 7 launches

    // Pre-additions in stored orientation: A quadrants are stored hm x hk (or hk x hm).
    const int64_t a_rows = transA ? hk : hm, a_cols = transA ? hm : hk;
    const int64_t b_rows = transB ? hn : hk, b_cols = transB ? hk : hn;
    auto grid2 = [&](int64_t rows, int64_t cols) {
        // 4 columns per thread on the (usual) 16-byte-aligned path
        int gx = static_cast<int>((cols + 1023) / 1024);
        if (gx > 32) gx = 32;
        int64_t gy = (int64_t)num_sms() * 8 / gx;
        if (gy > rows) gy = rows;
        if (gy > 65535) gy = 65535;
        if (gy < 1) gy = 1;
        return dim3(gx, static_cast<unsigned>(gy));
    };
    const int32_t* A11 = quad(A, lda, transA, hm, hk, 0, 0);
    const int32_t* A12 = quad(A, lda, transA, hm, hk, 0, 1);
    const int32_t* A21 = quad(A, lda, transA, hm, hk, 1, 0);
    const int32_t* A22 = quad(A, lda, transA, hm, hk, 1, 1);
    const int32_t* B11 = quad(B, ldb, transB, hk, hn, 0, 0);
    const int32_t* B12 = quad(B, ldb, transB, hk, hn, 0, 1);
    const int32_t* B21 = quad(B, ldb, transB, hk, hn, 1, 0);
    const int32_t* B22 = quad(B, ldb, transB, hk, hn, 1, 1);
    note_launch(2);
    preadd_kernel<<<grid2(a_rows, a_cols), 256, 0, st>>>(half.mp, 0, a_rows, a_cols, A11, A12, A21, A22, lda, S[0],
                                                         S[1], S[2], S[3]);
    preadd_kernel<<<grid2(b_rows, b_cols), 256, 0, st>>>(half.mp, 1, b_rows, b_cols, B11, B12, B21, B22, ldb, T[0],
                                                         T[1], T[2], T[3]);
    if (cudaGetLastError() != cudaSuccess) return FF_ERR_CUDA;

    // Product operands: (A side, ld), (B side, ld), in launch order P1, P2, P6, P7, P5,
    // P3, P4.  S/T temporaries are dense, stored orientation.
    const int32_t* aop[7] = {A11, A12, S[1], S[2], S[0], S[3], A22};
    const int64_t ald[7] = {lda, lda, a_cols, a_cols, a_cols, a_cols, lda};
    const int32_t* bop[7] = {B11, B21, T[1], T[2], T[0], B22, T[3]};
    const int64_t bld[7] = {ldb, ldb, b_cols, b_cols, b_cols, ldb, b_cols};
    for (int i = 0; i < 7; ++i) {
        if (launch_encode(half, transA ? 0 : 1, hm, hk, aop[i], ald[i], Al[i], st) != cudaSuccess) return FF_ERR_CUDA;
        if (launch_encode(half, transB ? 1 : 0, hn, hk, bop[i], bld[i], Bl[i], st) != cudaSuccess) return FF_ERR_CUDA;
    }

    int32_t* C11 = C;
    int32_t* C12 = C + hn;
    int32_t* C21 = C + hm * ldc;
    int32_t* C22 = C + hm * ldc + hn;
    // Schedule with two stored temporaries so that no product's epilogue updates
    // more than two quadrants (a slow epilogue holds the MMA back):
    //   P1 -> C11 <- a P1 + b C11,  T = P1                        (T stored raw)
    //   P2 -> C11 += a P2
    //   P6 -> U = P6 + T  (= U2 of App. A.2)                      (U stored raw)
    //   P7 -> C21 <- a (P7 + U) + b C21,  C22 <- a (P7 + U) + b C22
    //   P5 -> C12 <- a (P5 + U) + b C12,  C22 += a P5
    //   P3 -> C12 += a P3,   P4 -> C21 -= a P4
    // beta enters at the first write of each quadrant.
    int32_t* Tt = reinterpret_cast<int32_t*>(take(4 * hm * hn));
    int32_t* Ut = reinterpret_cast<int32_t*>(take(4 * hm * hn));
    const uint32_t p = half.mp.p, al = half.mp.alpha, be = half.mp.beta, nal = (p - al) % p;
    const OutSpec o1[2] = {{C11, al, be, 0, 0}, {Tt, 1, 0, hn, 0}};                    // P1
    const OutSpec o2[1] = {{C11, al, 1, 0, 0}};                                         // P2
    const OutSpec o6[1] = {{Ut, 1, 0, hn, 1}};                                          // P6 (+T)
    const OutSpec o7[2] = {{C21, al, be, 0, 1}, {C22, al, be, 0, 1}};                   // P7 (+U)
    const OutSpec o5[2] = {{C12, al, be, 0, 1}, {C22, al, 1, 0, 0}};                    // P5 (+U for C12)
    const OutSpec o3[1] = {{C12, al, 1, 0, 0}};                                         // P3
    const OutSpec o4[1] = {{C21, nal, 1, 0, 0}};                                        // P4
    const OutSpec* outs[7] = {o1, o2, o6, o7, o5, o3, o4};
    const int nouts[7] = {2, 1, 1, 2, 2, 1, 1};
    const int32_t* adds[7] = {nullptr, nullptr, Tt, Ut, Ut, nullptr, nullptr};
    for (int i = 0; i < 7; ++i) {
        const int e = launch_gemm_tc_multi(half, hm, hn, hk, Al[i], Bl[i], outs[i], nouts[i], ldc, i == 6 ? 1 : 0,
                                             scratch, st, adds[i], hn);
        if (e) return e;
    }
    return 0;
}

}  // namespace ff
