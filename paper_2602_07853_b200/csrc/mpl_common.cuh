// mpl_common.cuh — shared device/host definitions of the B200 MPM Lite library (sm_100a).
//
// Layout in HBM:
//   * 4^3-node blocks ("tiles") t = 0..T-1: every node block touched by an active cell block,
//     sorted by x-major block id.  Node vectors are tile-dense: node (t, l) at index t*64 + l,
//     l = (lx*4 + ly)*4 + lz.  Vector element = vec4<T> (x, y, z, pad).
//   * Cell block t shares the tile's coordinates; its structural cells are stored compactly
//     ("compact cells"), each tile's run padded to a multiple of 4 cells so every tile's tangent
//     block K[cs..ce) is 16-byte aligned for cp.async.bulk.
//   * Particles are kept sorted by (tile, base cell) after every resample.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>
#include <cstring>

#include "../../include/mpmlite.h"

#define MPL_MAXMAT 8

// Debug build (MPL_DEBUG=1 python -m paper_2602_07853_b200.build): device-side bounds checks that
// print the failing condition and trap (a stand-in for compute-sanitizer, which this pool closes).
#ifdef MPL_DEBUG
#include <cstdio>
#define DASSERT(c)                                                                                          \
    do {                                                                                                    \
        if (!(c)) {                                                                                         \
            printf("MPL_DEBUG assert failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__,   \
                   (int)blockIdx.x, (int)threadIdx.x);                                                      \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#define MPL_DEBUG_PRINT(ctx) fprintf(stderr, "[rank %d] %s\n", (ctx)->rank, (ctx)->err.c_str())
#else
#define MPL_DEBUG_PRINT(ctx) \
    do {                     \
    } while (0)
#define DASSERT(c) \
    do {           \
    } while (0)
#endif
#define MPL_MAXBOX 8
#define MPL_LOG_NEWTON 64

// ------------------------------------------------------------------------------------------
// vector types
// ------------------------------------------------------------------------------------------
struct __align__(16) f4 { float x, y, z, w; };
struct __align__(32) d4 { double x, y, z, w; };
template <class T> struct V4;
template <> struct V4<float> { typedef f4 type; };
template <> struct V4<double> { typedef d4 type; };
template <class T> using vec4 = typename V4<T>::type;

template <class T> __host__ __device__ __forceinline__ vec4<T> mk4(T x, T y, T z, T w) {
    vec4<T> r;
    r.x = x; r.y = y; r.z = z; r.w = w;
    return r;
}

// ------------------------------------------------------------------------------------------
// parameters passed by value to kernels
// ------------------------------------------------------------------------------------------
struct GridP {
    int n[3];          // cells per axis
    int nb[3];         // node-block (tile) coordinate extent per axis = n/4 + 1
    double dx, inv_dx;
    double origin[3];
};

struct MatP {
    int nmat;
    int kind[MPL_MAXMAT];  // 0 StVK-Hencky, 1 split Neo-Hookean, 2 J-based water (kappa = E)
    double mu[MPL_MAXMAT], lam[MPL_MAXMAT], rho[MPL_MAXMAT], kappa[MPL_MAXMAT];  // kappa = 2/3 mu + lam
    double sigy[MPL_MAXMAT];  // von Mises yield stress (kind 0; 0 = elastic)
    int plastic;              // any sigy > 0: fixed-point plasticity in Newton
};

struct BoxP {
    int nbox;
    double lo[MPL_MAXBOX][3], hi[MPL_MAXBOX][3], vel[MPL_MAXBOX][3];
};

// Tile geometry tables (device pointers)
struct TilesP {
    int T;                 // number of tiles (active node blocks)
    const int *coord;      // T*3 block coords
    const int *nbr_plus;   // T*8: tile at coord + o (o x-major in {0,1}^3) or -1
    const int *nbr_minus;  // T*8: tile at coord - o or -1
    const int *cell_start; // T+1: compact cell offsets (runs padded to multiples of 4)
    const uint8_t *cell_local; // C: local cell index 0..63, 0xFF = padding
    const int *cell_of;    // T*64: compact index of local cell or -1
    const int *tile_has_cells; // T: 1 if the cell block of this tile is active
};

// ------------------------------------------------------------------------------------------
// small math
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float mlog1p(float x) { return log1pf(x); }
__device__ __forceinline__ double mlog1p(double x) { return log1p(x); }
__device__ __forceinline__ float mexpm1(float x) { return expm1f(x); }
__device__ __forceinline__ double mexpm1(double x) { return expm1(x); }
__device__ __forceinline__ float msqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double msqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float mrsqrt(float x) { return rsqrtf(x); }
__device__ __forceinline__ double mrsqrt(double x) { return rsqrt(x); }
__device__ __forceinline__ float mabs(float x) { return fabsf(x); }
__device__ __forceinline__ double mabs(double x) { return fabs(x); }

// 3x3 row-major helpers (arrays fully unrolled into registers)
template <class T> __device__ __forceinline__ void mm3(const T A[9], const T B[9], T C[9]) {
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) C[3 * a + b] = A[3 * a] * B[b] + A[3 * a + 1] * B[3 + b] + A[3 * a + 2] * B[6 + b];
}
template <class T> __device__ __forceinline__ T det3(const T A[9]) {
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) + A[2] * (A[3] * A[7] - A[4] * A[6]);
}
// inverse-transpose B = A^{-T}, returns det
template <class T> __device__ __forceinline__ T inv_transpose3(const T A[9], T B[9]) {
    T c00 = A[4] * A[8] - A[5] * A[7], c01 = A[5] * A[6] - A[3] * A[8], c02 = A[3] * A[7] - A[4] * A[6];
    T c10 = A[2] * A[7] - A[1] * A[8], c11 = A[0] * A[8] - A[2] * A[6], c12 = A[1] * A[6] - A[0] * A[7];
    T c20 = A[1] * A[5] - A[2] * A[4], c21 = A[2] * A[3] - A[0] * A[5], c22 = A[0] * A[4] - A[1] * A[3];
    T det = A[0] * c00 + A[1] * c01 + A[2] * c02;
    T id = T(1) / det;
    // A^{-1}_{ab} = cof_{ba}/det  =>  A^{-T}_{ab} = cof_{ab}/det
    B[0] = c00 * id; B[1] = c01 * id; B[2] = c02 * id;
    B[3] = c10 * id; B[4] = c11 * id; B[5] = c12 * id;
    B[6] = c20 * id; B[7] = c21 * id; B[8] = c22 * id;
    return det;
}

// One Jacobi rotation zeroing S[p][q] of a symmetric 3x3 (NR convention), accumulating Q.
template <class T, int p, int q, int r>
__device__ __forceinline__ void jrot(T S[9], T Q[9]) {
    T apq = S[3 * p + q];
    if (apq == T(0)) return;
    T theta = (S[3 * q + q] - S[3 * p + p]) / (T(2) * apq);
    T t = T(1) / (mabs(theta) + msqrt(theta * theta + T(1)));
    t = theta < T(0) ? -t : t;
    T c = mrsqrt(t * t + T(1)), s = t * c;
    T app = S[3 * p + p] - t * apq, aqq = S[3 * q + q] + t * apq;
    T arp = S[3 * r + p], arq = S[3 * r + q];
    T nrp = c * arp - s * arq, nrq = s * arp + c * arq;
    S[3 * p + p] = app; S[3 * q + q] = aqq;
    S[3 * p + q] = S[3 * q + p] = T(0);
    S[3 * r + p] = S[3 * p + r] = nrp;
    S[3 * r + q] = S[3 * q + r] = nrq;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        T qp = Q[3 * a + p], qq = Q[3 * a + q];
        Q[3 * a + p] = c * qp - s * qq;
        Q[3 * a + q] = s * qp + c * qq;
    }
}

// Symmetric eigen-decomposition by cyclic Jacobi: A = Q diag(w) Q^T (columns of Q).
template <class T> __device__ __forceinline__ void sym_eig3(const T A[9], T w[3], T Q[9]) {
    T S[9];
#pragma unroll
    for (int a = 0; a < 9; a++) { S[a] = A[a]; Q[a] = (a % 4 == 0) ? T(1) : T(0); }
    const int maxsweep = sizeof(T) == 4 ? 6 : 10;
    const T tol = sizeof(T) == 4 ? T(1e-14) : T(1e-30);
    for (int sw = 0; sw < maxsweep; sw++) {
        T off = S[1] * S[1] + S[2] * S[2] + S[5] * S[5];
        T dia = S[0] * S[0] + S[4] * S[4] + S[8] * S[8];
        if (!(off > tol * dia)) break;
        jrot<T, 0, 1, 2>(S, Q);
        jrot<T, 0, 2, 1>(S, Q);
        jrot<T, 1, 2, 0>(S, Q);
    }
    w[0] = S[0]; w[1] = S[4]; w[2] = S[8];
}

// Divided difference of log (Daleckii-Krein), from eigenvalues lx = x-1, ly = y-1 of b - I (amb-20)
template <class T> __device__ __forceinline__ T dlog(T lx, T ly) {
    T y = T(1) + ly;
    T t = (lx - ly) / y;
    const T thr = sizeof(T) == 4 ? T(2e-2) : T(1e-3);
    if (mabs(t) < thr) return (T(1) + t * (T(-0.5) + t * (T(1) / T(3) + t * (T(-0.25) + t * T(0.2))))) / y;
    return mlog1p(t) / (lx - ly);
}

// ---- split Neo-Hookean (PAPER §4.3.2) in forms that keep fp32 accurate at small strain:
// with H = F - I and Bm = b - I = H + H^T + H H^T,
//   J - 1 = tr H + (tr(H)^2 - tr(H^2))/2 + det H,   J^{-2/3} - 1 = expm1(-2/3 log1p(J - 1)),
//   tau = mu J^{-2/3} dev(Bm) + kappa/2 (J-1)(J+1) I                      (Eq. split-nh-tau),
//   Psi = mu/2 (3 (J^{-2/3}-1) + tr(Bm) J^{-2/3}) + kappa/4 f(J-1),
//   f(x) = x (2 + x) - 2 log1p(x)                                         (Eq. split-nh-energy).
template <class T> __device__ __forceinline__ T det_ipm1(const T H[9]) {  // det(I + H) - 1
    const T tr = H[0] + H[4] + H[8];
    const T tr2 = H[0] * H[0] + H[4] * H[4] + H[8] * H[8] + T(2) * (H[1] * H[3] + H[2] * H[6] + H[5] * H[7]);
    return tr + T(0.5) * (tr * tr - tr2) + det3(H);
}
// Von Mises return map in Hencky strain space (P:658-663 fixed-point plasticity), as a right
// factor F^E = F P with P = V diag(exp((s - 1) e_dev)) V^T from C = F^T F = V sigma^2 V^T, e = log sigma,
// s = sqrt(2/3) sigma_y / (2 mu |e_dev|) when 2 mu |e_dev| > sqrt(2/3) sigma_y (else P = I).  Takes
// H = F - I, returns P - I (cancellation-free: C - I = H + H^T + H^T H, e = log1p(.)/2, expm1).
template <class T> __device__ __forceinline__ bool vm_plastic_Pm1(const T H[9], T mu, T sigy, T Pm1[9]) {
    T Cm[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            Cm[3 * a + b] = H[3 * a + b] + H[3 * b + a] + H[a] * H[b] + H[3 + a] * H[3 + b] + H[6 + a] * H[6 + b];
    T lam[3], V[9];
    sym_eig3(Cm, lam, V);
    const T e0 = T(0.5) * mlog1p(lam[0]), e1 = T(0.5) * mlog1p(lam[1]), e2 = T(0.5) * mlog1p(lam[2]);
    const T m3 = (e0 + e1 + e2) / T(3);
    const T d0 = e0 - m3, d1 = e1 - m3, d2 = e2 - m3;
    const T nrm = msqrt(d0 * d0 + d1 * d1 + d2 * d2);
    const T ry = T(0.81649658092772603) * sigy;  // sqrt(2/3) sigma_y
#pragma unroll
    for (int a = 0; a < 9; a++) Pm1[a] = T(0);
    if (!(T(2) * mu * nrm > ry)) return false;
    const T sm1 = ry / (T(2) * mu * nrm) - T(1);
    const T q0 = mexpm1(sm1 * d0), q1 = mexpm1(sm1 * d1), q2 = mexpm1(sm1 * d2);
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            Pm1[3 * a + b] = V[3 * a] * V[3 * b] * q0 + V[3 * a + 1] * V[3 * b + 1] * q1 + V[3 * a + 2] * V[3 * b + 2] * q2;
    return true;
}

template <class T> __device__ __forceinline__ T nh_f(T x) {  // x (2 + x) - 2 log1p(x), series near 0
    // the series (truncation ~x^8/4) replaces the cancelling direct form below |x| = 0.1 (fp32) / 1e-3 (fp64)
    if (mabs(x) < (sizeof(T) == 4 ? T(0.1) : T(1e-3))) {
        // 2 x^2 - 2/3 x^3 + 1/2 x^4 - 2/5 x^5 + 1/3 x^6 - 2/7 x^7
        return x * x * (T(2) + x * (T(-2.0 / 3.0) + x * (T(0.5) + x * (T(-0.4) + x * (T(1.0 / 3.0) + x * T(-2.0 / 7.0))))));
    }
    return x * (T(2) + x) - T(2) * mlog1p(x);
}

// Programmatic dependent launch (PCG loop): a kernel launched with launch_pdl may be scheduled while
// the previous kernel on the stream drains; every such kernel calls pdl_trigger() and then pdl_wait()
// before touching any memory, so it only overlaps the previous kernel's tail / its own launch latency.
// Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();  // MPL_PDL (default on)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    if (!pdl_enabled()) {
        k<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Warp-cooperative AoS transfers for the particle kernels: the warp's 32 consecutive particles p0 ..
// p0 + 31 (p0 % 32 == 0) own W contiguous reals each at A + W p0; 16-byte loads / stores of the whole
// 32 W-real block through a per-warp shared buffer `sm` (>= 32 W reals), then each lane reads / writes
// its W reals there (odd W: conflict-free).  One 16-byte access per lane per 4 / W particles instead of
// W scalar accesses per particle.  All 32 lanes must call.
template <class T, int W>
__device__ __forceinline__ void warp_load_aos(const T *__restrict__ A, int64_t p0, T *sm, T out[W]) {
    const int lane = threadIdx.x & 31;
    constexpr int NV = (int)(32 * W * sizeof(T) / 16);
    const float4 *src = reinterpret_cast<const float4 *>(A + (int64_t)W * p0);
    float4 *d = reinterpret_cast<float4 *>(sm);
#pragma unroll
    for (int i = lane; i < NV; i += 32) d[i] = src[i];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < W; a++) out[a] = sm[lane * W + a];
    __syncwarp();
}
template <class T, int W>
__device__ __forceinline__ void warp_store_aos(T *__restrict__ A, int64_t p0, T *sm, const T in[W]) {
    const int lane = threadIdx.x & 31;
    constexpr int NV = (int)(32 * W * sizeof(T) / 16);
#pragma unroll
    for (int a = 0; a < W; a++) sm[lane * W + a] = in[a];
    __syncwarp();
    float4 *dst = reinterpret_cast<float4 *>(A + (int64_t)W * p0);
    const float4 *s4 = reinterpret_cast<const float4 *>(sm);
#pragma unroll
    for (int i = lane; i < NV; i += 32) dst[i] = s4[i];
    __syncwarp();
}

// symmetric 9x9 upper-triangle packing: row r (r = 3a+b) stores s = r..8
__host__ __device__ __forceinline__ constexpr int kofs(int r) { return r * 9 - (r * (r - 1)) / 2; }
__host__ __device__ __forceinline__ constexpr int kidx(int r, int s) { return kofs(r) + (s - r); }

// warp/block reductions (double).  Cross-CTA sums go to NSTRIPE "striped" accumulators
// (one fp64 atomic per CTA into stripe blockIdx % NSTRIPE): tens of thousands of same-address
// atomics per launch serialise in L2, striping removes that contention.
#define NSTRIPE 32
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// all threads of the block must call; adds the block total into acc[blockIdx.x % NSTRIPE]
__device__ __forceinline__ void block_add(double v, double *acc) {
    __shared__ double red_[32];
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red_[w] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double x = threadIdx.x < nw ? red_[threadIdx.x] : 0.0;
        x = warp_sum(x);
        if (threadIdx.x == 0 && x != 0.0) atomicAdd(&acc[blockIdx.x % NSTRIPE], x);
    }
}
// sum of NSTRIPE stripes, broadcast to the block (all threads must call)
__device__ __forceinline__ double stripe_sum_bcast(const double *acc) {
    __shared__ double s_;
    if (threadIdx.x < 32) {
        double x = acc[threadIdx.x];
        x = warp_sum(x);
        if (threadIdx.x == 0) s_ = x;
    }
    __syncthreads();
    double r = s_;
    __syncthreads();
    return r;
}
inline double host_stripes(const double *h) {
    double s = 0;
    for (int i = 0; i < NSTRIPE; i++) s += h[i];
    return s;
}

// Tangent layout (per tile, ncp = padded cell count): element e < NCH*VEC of cell j at
// base + ((e / VEC) * ncp + j) * VEC + e % VEC  (16-byte vectors, coalesced across cells);
// the remaining element (e = 44) at base + NCH*VEC*ncp + j.  base = cstart[t] * 45.
template <class T> struct KL {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int NCH = 45 / VEC;
    static constexpr int REM = 45 - NCH * VEC;
};
// Tangent layout per tile: n = the tile's real cells (no padding), block of 45 n reals (rounded up
// to 4) at t_kstart[t], chunked as k_off with ncp = n.  Slot order: k_hvp_wz's "kz" order (layout 1:
// the cell at local position l = 16 lx + 4 ly + lz is ranked by kz_key(l) = the wz lane (16 (lz >> 1) +
// 4 lx + ly) for even lz, 32 + that lane for odd lz, so a warp's 16-byte loads of one chunk are
// contiguous), or the natural compact order (layout 3: slot = rank of l; k_hvp_wh).
__host__ __device__ __forceinline__ constexpr int kz_key(int l) {
    return ((l & 1) << 5) | (((l >> 1) & 1) << 4) | ((l >> 4) << 2) | ((l >> 2) & 3);
}
// compressed tangent (fp32, k_hvp_wz): KC_REALS reals per cell (q_U's x, y, z 3, W = S V 9,
// c psi 6, c (a, b) 6), per tile one pair slot per wz lane holding a cell, 2 KC_REALS reals per slot
constexpr int KC_REALS = 24;
int hvp_kz_layout(int precision);  // 1: compact kz order (k_hvp_wz), 3: natural compact order (k_hvp_wh)
int hvp_variant();                 // fp32 HVP kernel: 0 k_hvp_wz, 1 k_hvp_wh
template <class T> __host__ __device__ __forceinline__ int64_t k_off(int64_t base, int ncp, int j, int e) {
    return e < KL<T>::NCH * KL<T>::VEC
               ? base + ((int64_t)(e / KL<T>::VEC) * ncp + j) * KL<T>::VEC + (e % KL<T>::VEC)
               : base + (int64_t)KL<T>::NCH * KL<T>::VEC * ncp + (int64_t)j * KL<T>::REM + (e - KL<T>::NCH * KL<T>::VEC);
}

// ------------------------------------------------------------------------------------------
// host-side context
// ------------------------------------------------------------------------------------------
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};

// Per-Newton-iteration PCG accumulators (one slot per CG iteration; fp64)
struct CGSlot {
    double rz[NSTRIPE];   // r_j . z_j   (striped)
    double rr[NSTRIPE];   // r_j . r_j
    double pHp[NSTRIPE];  // p_j . H p_j  (single-reduction PCG: u_j . H u_j)
    double alpha, pad;    // single-reduction PCG: the step alpha_j, written by iteration j's vector kernel
};

// device-side scalar block (fp64 accumulators and flags)
struct DevScalars {
    double energy[NSTRIPE];  // Phi accumulator (striped)
    double inv_any;          // 1.0 if det(I + dt G) <= 0 was seen (reduced with energy; amb-21)
    double gnorm2[NSTRIPE];  // ||g_free||^2
    double gp[NSTRIPE];      // g . p
    int nonfinite;
    int oob_particle;  // min index of an out-of-domain particle (INT_MAX = none)
    int inv_particle;  // min index of an inverted particle
    int neg_curv;      // PCG breakdown (p.Hp <= 0)
    int cg_done_iter;  // first iteration index at which PCG converged (or -1)
    int cg_j[2];       // graph-captured PCG (MPL_PCG_GRAPH): iteration index read by the kernels of an even /
                       // odd iteration, advanced on the device by its update2
    double cg_thr;     // graph-captured PCG: the convergence threshold of the current Newton iteration
};

// Communicator between the slab ranks.  Every method is collective over the ranks and
// stream-ordered on ctx->stream; implementations: NCCL (one process per GPU, mpl_comm.cu) and an
// in-process loopback group (ranks as host threads of one process, for single-GPU testing).
struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() {}
    // in-place sum of n doubles (device memory) over all ranks; every rank gets the same values
    virtual mpl_status allreduce(mpl_ctx ctx, double *dev, int64_t n) = 0;
    // neighbour exchange: send_lo -> rank-1 (arrives in its recv_hi), send_hi -> rank+1 (its recv_lo).
    // Byte counts must match pairwise; a missing neighbour's arguments are ignored.
    virtual mpl_status neighbors(mpl_ctx ctx, const void *send_lo, size_t n_send_lo, void *recv_lo, size_t n_recv_lo,
                                 const void *send_hi, size_t n_send_hi, void *recv_hi, size_t n_recv_hi) = 0;
};

struct mpl_ctx_s {
    int precision = 32, device = 0, rank = 0, nranks = 1;
    Comm *comm = nullptr;                  // nranks > 1
    int slab_lo = 0, slab_hi = 1 << 30;    // owned cell-block x range [slab_lo, slab_hi) (4-cell blocks)
    std::vector<int> cuts;                 // nranks + 1 slab boundaries (cell blocks)
    int64_t np_own = 0;                    // owned particles (the rest of np are ghosts, pid < 0)
    DevBuf pv_alt, pG_alt;                 // redistribution targets for v, G
    DevBuf mig_send_lo, mig_send_hi, mig_recv_lo, mig_recv_hi, mig_cnt;
    DevBuf pl_send_lo, pl_send_hi, pl_recv_lo, pl_recv_hi;  // compact interface-face halo buffers
    // Interface faces: this rank's tiles on the lower / upper shared node-block planes,
    // sorted by (by, bz); the neighbour's list in the same order arrives once per resample and is matched
    // to local tiles (map: received entry -> local tile or -1).  A halo message is 16 nodes per listed tile.
    DevBuf t_lo_list, t_hi_list, t_lo_map, t_hi_map;
    int n_lo_tiles = 0, n_hi_tiles = 0, n_lo_recv = 0, n_hi_recv = 0;
    // the HVP split for overlap: tiles whose cells or owned nodes touch a shared node plane (node-block x in
    // {slab_lo - 1, slab_lo, slab_hi - 1, slab_hi}) first, then the interior tiles
    DevBuf t_bnd, t_int;
    int n_bnd = 0, n_int = 0;
    cudaStream_t hstream = nullptr;     // halo stream of the overlapped HVP (NCCL transport)
    cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
    DevBuf n_own, n_mown;                  // per node: owner flag (uint8), owned mass (m if owner else 0)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // pinned staging for the solver's small device->host control reads (counts, CG scalars): a copy
    // into pageable memory waits behind any large D2H in flight on another stream (measured: 26 ms
    // behind a 1.5 GB readback), a copy into pinned memory does not (0.07 ms)
    char *pio_buf = nullptr;  // mapped pinned host memory; pio_dev: its device address
    char *pio_dev = nullptr;
    size_t pio_cap = 0, pio_used = 0;
    struct PioPend { void *dst; size_t off, n; };
    std::vector<PioPend> pio_pend;
    // pipelined particle I/O (mpl_stage_particles / mpl_get_particles_async): copy stream + events,
    // a staged input set adopted by the next resample, a readback set copied out on the copy stream
    cudaStream_t cstream = nullptr, rstream = nullptr;  // H2D staging / D2H readback (separate DMA engines)
    cudaEvent_t ev_staged = nullptr, ev_adopted = nullptr, ev_rb_ready = nullptr, ev_rb_done = nullptr;
    bool staged = false, adopted_once = false, rb_once = false;
    int64_t staged_n = 0;
    DevBuf sx, sv, sF, sG, svol, smat;  // staged inputs (swapped with the live set on adoption)
    DevBuf rb[4];                       // readback: x, v, F, G in input order
    std::string err;

    GridP grid{};
    MatP mats{};
    BoxP boxes{};
    double gravity[3] = {0.0, -9.81, 0.0};
    double dt = 0.0;

    // particles (sorted layout; ping-pong A/B)
    int64_t np = 0;
    int cur = 0;  // which particle buffer set is current
    DevBuf px[2], pF[2], pv, pG, pvol[2], pmat[2], pid[2];
    DevBuf pkey, prank, prec, pbase, pskey;  // per-particle scratch; pskey/prec in sorted order
    DevBuf psrc;                             // sort as a gather: source particle of each sorted slot
    // k_scatter sorts x, F, vol, mat, pid (ping-pong sets) but not v and G: P2Q reads them through the
    // record and G2P rewrites them in sorted order.  Between the two, v / G still follow the previous
    // order; vg_unsorted records that, and sync_vg_order (a gather through the resample's sort map
    // pkey / prank / t_bstart) restores one order before anything else reads v / G (a second resample,
    // mpl_get_particles*).
    bool vg_unsorted = false;
    // Hessian mode of the cached tangent: psd_default (mpl_set_psd_projection) for mpl_linearize,
    // psd_now = the value the current linearisation uses (newton_impl sets it from its solver cfg)
    int psd_default = 0, psd_now = 0;
    // compressed tangent: cells with more than one occupied material slot (from the resample)
    // and the format the last full linearisation wrote (0: 45-number K, 1: compressed, 28 reals per cell)
    int64_t multi_slot_cells = 0;
    int64_t nonid_base_cells = 0;  // cells with an occupied slot whose base S is not I (E != 0)
    int kc_now = 0;

    // tiles
    int T = 0;
    int64_t C = 0;  // compact cells incl. padding
    int64_t n_cells_active = 0, n_nodes_active = 0, n_blocks_active = 0, n_free_nodes = 0;
    int64_t launches = 0;  // kernels launched by this context (cumulative)
    int dense_n = 0;  // nb0*nb1*nb2
    DevBuf cflag, nflag, tile_of, scan_tmp;
    DevBuf t_coord, t_nplus, t_nminus, t_cstart, t_ccount, t_hascells, t_bcount, t_bstart, t_cellof, t_cmask, t_perm;
    DevBuf t_ncell, t_kcnt, t_kstart;  // real cells per tile; tangent reals per tile (rounded to 4) and offsets
    DevBuf t_kcnt2, t_kstart2;         // the same for the compressed tangent (56 reals per pair slot)
    DevBuf c_local;
    // quadrature (compact cells)
    DevBuf q_m, q_mv, q_mG, q_slot;  // q_slot: C * nmat * 16 (V, E xx yy zz xy yz xz, tau (6), pad)
    DevBuf q_Sp;                     // plastic runs: C * nmat * 9, S_k - I of the current Newton iterate
    DevBuf q_vc;                     // load: (v_c, G_c) per cell, 12 reals
    DevBuf K;                        // tangent (scaled by 1/(16 dx^2)), per tile at t_kstart, 45 reals per real cell
    // nodes (tile-dense, T*64)
    DevBuf n_mass, n_flag, n_vn, n_vhat, n_v, n_vt, n_g, n_diag, n_invD, n_x, n_r, n_p, n_Hp, n_u, n_u2, n_act;
    // canonical node index per tile-dense node (-1 inactive)
    DevBuf n_canon, n_list;  // n_list: canonical -> tile-dense index
    DevBuf n_ps;             // single-reduction PCG: p and s (= H p) compact SoA, 6 x SA reals
    DevBuf scalars, cg_slots, io_stage, io_stage2;
    int cg_slot_cap = 0;
    DevBuf host_pinned;  // small pinned staging
    bool have_particles = false, resampled = false, linearized = false, solved = false;
    std::vector<cudaEvent_t> ev;
};

// ------------------------------------------------------------------------------------------
// error helpers
// ------------------------------------------------------------------------------------------
#define MPL_CUDA(call)                                                                  \
    do {                                                                                \
        const cudaError_t mpl_cuda_err_ = (call);                                       \
        if (mpl_cuda_err_ != cudaSuccess) {                                             \
            ctx->err = std::string("CUDA error: ") + cudaGetErrorString(mpl_cuda_err_) + \
                       " at " +                                                         \
                       __FILE__ + ":" + std::to_string(__LINE__);                       \
            MPL_DEBUG_PRINT(ctx);                                                       \
            return MPL_ERR_CUDA;                                                        \
        }                                                                               \
    } while (0)

#define MPL_CHECK(st)                                      \
    do {                                                   \
        const mpl_status mpl_check_st_ = (st);             \
        if (mpl_check_st_ != MPL_OK) return mpl_check_st_; \
    } while (0)

mpl_status ensure(mpl_ctx ctx, DevBuf &b, size_t bytes);
// every device buffer of a context with its name (destroy, debug guard checks)
// Enqueue a small device->host read into the context's pinned staging; the destination is filled by
// the next d2h_sync (stream synchronisation + host copy).
inline mpl_status d2h_sync(mpl_ctx ctx, cudaStream_t st) {
    MPL_CUDA(cudaStreamSynchronize(st));
    for (auto &q : ctx->pio_pend) memcpy(q.dst, ctx->pio_buf + q.off, q.n);
    ctx->pio_pend.clear();
    ctx->pio_used = 0;
    return MPL_OK;
}
// Small device->host reads (counts, CG scalars, slot histories) are written by a kernel straight
// into mapped pinned host memory instead of a cudaMemcpyAsync: a DMA copy on the compute stream queued
// behind the pipelined 1.5 GB particle readback on the copy engine (cfg4: the resample's first count
// read waited ~29 ms for it), a kernel store over the host link does not.
static __global__ void k_pio_copy(char *__restrict__ dst, const char *__restrict__ src, size_t n) {
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n; i += (size_t)gridDim.x * blockDim.x * 16) {
        if (i + 16 <= n && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
            *reinterpret_cast<uint4 *>(dst + i) = *reinterpret_cast<const uint4 *>(src + i);
        } else {
            for (size_t j = i; j < i + 16 && j < n; j++) dst[j] = src[j];
        }
    }
}
inline mpl_status d2h(mpl_ctx ctx, void *dst, const void *src, size_t n, cudaStream_t st) {
    size_t off = (ctx->pio_used + 15) & ~(size_t)15;
    if (off + n > ctx->pio_cap) {
        if (!ctx->pio_pend.empty()) MPL_CHECK(d2h_sync(ctx, st));
        size_t cap = ctx->pio_cap * 2 > n ? ctx->pio_cap * 2 : n;
        if (cap < ((size_t)1 << 16)) cap = (size_t)1 << 16;
        if (ctx->pio_buf) cudaFreeHost(ctx->pio_buf);
        ctx->pio_buf = nullptr;
        ctx->pio_dev = nullptr;
        MPL_CUDA(cudaHostAlloc((void **)&ctx->pio_buf, cap, cudaHostAllocMapped));
        MPL_CUDA(cudaHostGetDevicePointer((void **)&ctx->pio_dev, ctx->pio_buf, 0));
        ctx->pio_cap = cap;
        off = 0;
    }
    if (n) {
        const size_t chunks = (n + 15) / 16;
        const unsigned blocks = (unsigned)(chunks < 256 ? 1 : (chunks / 256 < 1024 ? chunks / 256 + 1 : 1024));
        k_pio_copy<<<blocks, 256, 0, st>>>(ctx->pio_dev + off, static_cast<const char *>(src), n);
        MPL_CUDA(cudaGetLastError());
    }
    ctx->pio_pend.push_back({dst, off, n});
    ctx->pio_used = off + n;
    return MPL_OK;
}

template <class F> void for_each_buf(mpl_ctx ctx, F f) {
    struct NB { const char *name; DevBuf &b; };
    NB all[] = {
        {"sx", ctx->sx},
        {"sv", ctx->sv},
        {"sF", ctx->sF},
        {"sG", ctx->sG},
        {"svol", ctx->svol},
        {"smat", ctx->smat},
        {"rb[0]", ctx->rb[0]},
        {"rb[1]", ctx->rb[1]},
        {"rb[2]", ctx->rb[2]},
        {"rb[3]", ctx->rb[3]},
        {"px[0]", ctx->px[0]},
        {"px[1]", ctx->px[1]},
        {"pF[0]", ctx->pF[0]},
        {"pF[1]", ctx->pF[1]},
        {"pv", ctx->pv},
        {"pG", ctx->pG},
        {"pvol[0]", ctx->pvol[0]},
        {"pvol[1]", ctx->pvol[1]},
        {"pmat[0]", ctx->pmat[0]},
        {"pmat[1]", ctx->pmat[1]},
        {"pid[0]", ctx->pid[0]},
        {"pid[1]", ctx->pid[1]},
        {"pkey", ctx->pkey},
        {"prank", ctx->prank},
        {"prec", ctx->prec},
        {"pbase", ctx->pbase},
        {"pskey", ctx->pskey},
        {"cflag", ctx->cflag},
        {"nflag", ctx->nflag},
        {"tile_of", ctx->tile_of},
        {"scan_tmp", ctx->scan_tmp},
        {"t_coord", ctx->t_coord},
        {"t_nplus", ctx->t_nplus},
        {"t_nminus", ctx->t_nminus},
        {"t_cstart", ctx->t_cstart},
        {"t_ccount", ctx->t_ccount},
        {"t_hascells", ctx->t_hascells},
        {"t_bcount", ctx->t_bcount},
        {"t_bstart", ctx->t_bstart},
        {"t_cellof", ctx->t_cellof},
        {"t_cmask", ctx->t_cmask},
        {"t_perm", ctx->t_perm},
        {"c_local", ctx->c_local},
        {"q_m", ctx->q_m},
        {"q_mv", ctx->q_mv},
        {"q_mG", ctx->q_mG},
        {"q_slot", ctx->q_slot},
        {"q_Sp", ctx->q_Sp},
        {"q_vc", ctx->q_vc},
        {"K", ctx->K},
        {"t_ncell", ctx->t_ncell},
        {"t_kcnt", ctx->t_kcnt},
        {"t_kstart", ctx->t_kstart},
        {"t_kcnt2", ctx->t_kcnt2},
        {"t_kstart2", ctx->t_kstart2},
        {"n_mass", ctx->n_mass},
        {"n_flag", ctx->n_flag},
        {"n_vn", ctx->n_vn},
        {"n_vhat", ctx->n_vhat},
        {"n_v", ctx->n_v},
        {"n_vt", ctx->n_vt},
        {"n_g", ctx->n_g},
        {"n_diag", ctx->n_diag},
        {"n_invD", ctx->n_invD},
        {"n_x", ctx->n_x},
        {"n_r", ctx->n_r},
        {"n_p", ctx->n_p},
        {"psrc", ctx->psrc},
        {"n_ps", ctx->n_ps},
        {"n_Hp", ctx->n_Hp},
        {"n_u", ctx->n_u},
        {"n_u2", ctx->n_u2},
        {"n_act", ctx->n_act},
        {"n_canon", ctx->n_canon},
        {"n_list", ctx->n_list},
        {"scalars", ctx->scalars},
        {"cg_slots", ctx->cg_slots},
        {"io_stage", ctx->io_stage},
        {"io_stage2", ctx->io_stage2},
        {"pv_alt", ctx->pv_alt},
        {"pG_alt", ctx->pG_alt},
        {"mig_send_lo", ctx->mig_send_lo},
        {"mig_send_hi", ctx->mig_send_hi},
        {"mig_recv_lo", ctx->mig_recv_lo},
        {"mig_recv_hi", ctx->mig_recv_hi},
        {"mig_cnt", ctx->mig_cnt},
        {"pl_send_lo", ctx->pl_send_lo},
        {"pl_send_hi", ctx->pl_send_hi},
        {"pl_recv_lo", ctx->pl_recv_lo},
        {"pl_recv_hi", ctx->pl_recv_hi},
        {"t_lo_list", ctx->t_lo_list},
        {"t_hi_list", ctx->t_hi_list},
        {"t_lo_map", ctx->t_lo_map},
        {"t_hi_map", ctx->t_hi_map},
        {"t_bnd", ctx->t_bnd},
        {"t_int", ctx->t_int},
        {"n_own", ctx->n_own},
        {"n_mown", ctx->n_mown}
    };
    for (NB &x : all) f(x.name, x.b);
}
mpl_status debug_check_guards(mpl_ctx ctx, const char *where);
#ifdef MPL_DEBUG
#define DBG_GUARDS(where) MPL_CHECK(debug_check_guards(ctx, where))
#else
#define DBG_GUARDS(where) \
    do {                  \
    } while (0)
#endif


// kernels' host launchers (defined in k_*.cu), templated on the compute precision
template <class T> mpl_status resample_impl(mpl_ctx ctx, double dt);
template <class T> mpl_status linearize_impl(mpl_ctx ctx, const void *v_tile, int mode, double *phi);
template <class T> mpl_status hvp_tile(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *pHp_accum);
template <class T> mpl_status launch_hvp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu,
                                         const CGSlot *cgs, int cgj, double cgthr, const int *tlist = nullptr,
                                         int ntl = 0, const int *jdev = nullptr);
template <class T> mpl_status newton_impl(mpl_ctx ctx, const mpl_solver_cfg *cfg, mpl_solve_stats *st);
template <class T> mpl_status g2p_impl(mpl_ctx ctx, double dt);
template <class T> mpl_status sync_vg_order(mpl_ctx ctx);
template <class T> mpl_status explicit_impl(mpl_ctx ctx);

template <class T> mpl_status stage_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F,
                                              const void *G, const void *vol, const int32_t *mat);
template <class T> mpl_status adopt_staged(mpl_ctx ctx);
template <class T> mpl_status export_particles_async(mpl_ctx ctx, void *x, void *v, void *F, void *G);
mpl_status io_streams(mpl_ctx ctx);
template <class T> mpl_status canon_to_tile(mpl_ctx ctx, const void *src, void *dst_tile);
template <class T> mpl_status tile_to_canon(mpl_ctx ctx, const void *src_tile, void *dst);
template <class T> mpl_status export_quadrature(mpl_ctx ctx, int32_t *ijk, void *m_c, void *v_c, void *G_c,
                                                void *V_ck, void *tau_ck, void *S_ck);
template <class T> mpl_status export_particles(mpl_ctx ctx, void *x, void *v, void *F, void *G);
// multi-rank plumbing (mpl_comm.cu)
template <class T> mpl_status redistribute_particles(mpl_ctx ctx);
template <class T> mpl_status halo_sum_nodes(mpl_ctx ctx, void *a_tile, void *b_tile);
bool comm_is_nccl(mpl_ctx ctx);
template <class T> mpl_status ghost_nodes_from_upper(mpl_ctx ctx, void *v_tile);
template <class T> mpl_status c2n_halo(mpl_ctx ctx);
template <class T> mpl_status export_owned_particles(mpl_ctx ctx, void *x, void *v, void *F, void *G, int32_t *ids,
                                                     int32_t *base_ijk);
mpl_status build_interface_lists(mpl_ctx ctx);
mpl_status debug_check_tiles(mpl_ctx ctx, const char *where);
mpl_status allreduce_d(mpl_ctx ctx, double *dev, int64_t n);
mpl_status agree(mpl_ctx ctx, mpl_status local);
inline bool multi(mpl_ctx ctx) { return ctx->nranks > 1; }
bool serial_mode();
struct ApiLock {  // MPL_LOOPBACK_SERIAL debugging aid (mpl_api.cu)
    bool on;
    ApiLock();
    ~ApiLock();
};
int api_lock_release_all();
void api_lock_reacquire(int depth);
// lumped mass counted by this rank (m_i on owned nodes, 0 on the copies of shared nodes)
inline const void *owned_mass(mpl_ctx ctx) { return multi(ctx) ? ctx->n_mown.p : ctx->n_mass.p; }
mpl_status comm_create(mpl_ctx ctx, const mpl_config *cfg);
void comm_destroy(mpl_ctx ctx);

template <class T> mpl_status import_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F,
                                               const void *G, const void *vol, const int32_t *mat);

enum { LIN_ENERGY = 0, LIN_GRAD = 1, LIN_FULL = 2 };
