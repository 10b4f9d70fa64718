// k_hvp.cu — SURVEY §8(a) row a6, the graded kernel: the matrix-free Hessian-vector product
//     (H u)_i = m_i u_i + sum_{c ∋ i} (K_c : dG_c(u)) grad w_ic ,   dG_c(u) = sum_j u_j (x) grad w_jc
// (App. B: H = M + d^2 E/dv^2; grad w_ic = (x_i - x_c)/(2 dx^2); "matrix-free
// PCG" P:495), with K_c the cached 9x9 symmetric tangent of the quadrature point (k_linearize).
//
// Two kernels (the fourteen variants measured slower in round 1 are described in DESIGN.md
// §5 "history" and were removed from the library):
//   k_hvp_wz (fp32 default): one warp per 4^3 tile, two z-adjacent cells per lane, tangent of the next
//     tile prefetched into registers with L2 evict-first streaming loads, u halo cp.async double-buffered;
//   k_hvp_wh (fp64 default, MPL_HVP_KERNEL=wh for fp32): one warp per half tile, one cell per lane.
// u . Hu = sum_i m_i |u_i|^2 + sum_c dG:K:dG is accumulated exactly (striped fp64 accumulators); it is
// p^T H p of the PCG step.
#include <cstdlib>

#include "mpl_common.cuh"

namespace {

__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

template <class T> __device__ __forceinline__ void atomic_add3(vec4<T> *p, T x, T y, T z);
template <> __device__ __forceinline__ void atomic_add3<float>(f4 *p, float x, float y, float z) {
    atomicAdd(reinterpret_cast<float4 *>(p), make_float4(x, y, z, 0.f));
}
template <> __device__ __forceinline__ void atomic_add3<double>(d4 *p, double x, double y, double z) {
    atomicAdd(&p->x, x);
    atomicAdd(&p->y, y);
    atomicAdd(&p->z, z);
}

// ---- cp.async (LDGSTS) ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16s(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4s(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ f4 lds4(uint32_t a) {
    f4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds1(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts4z(uint32_t a) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(a), "f"(0.f) : "memory");
}
__device__ __forceinline__ void sts1z(uint32_t a) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(0.f) : "memory"); }
template <class T> __device__ __forceinline__ void cp_async_real(T *dst, const T *src);
template <> __device__ __forceinline__ void cp_async_real<float>(float *dst, const float *src) { cp_async4(dst, src); }
template <> __device__ __forceinline__ void cp_async_real<double>(double *dst, const double *src) { cp_async8(dst, src); }
// ---------------------------------------------------------------------------------------------
// k_hvp_wz (fp32 default): one warp per tile, two z-adjacent cells per lane, no block barriers.
//   * lane = 16 zp + 4 lx + ly owns cells A = (lx, ly, 2zp) and B = (lx, ly, 2zp + 1); they share the
//     4 nodes of the plane z = 2zp + 1, so the lane reads 12 node vectors instead of 16 and scatters
//     into 12 nodes instead of 16;
//   * dG of both cells by tensor-product sums per node plane (7 adds per plane and component);
//   * corner forces from 4 distinct sums per component and cell, signs folded into the adds;
//   * the tangent uses the "kz" slot order (kz_key): the A cells of a tile first, then the B cells,
//     each in lane order, so a warp's 16-byte loads of one chunk are contiguous; the 90 tangent
//     numbers of the next tile are loaded (L2 evict-first) as soon as the current tile's K dG is done;
//   * the u halo (shared slot 5x + 26y + z: conflict-free 16-byte accesses for every quarter-warp)
//     and the owned masses are cp.async double-buffered per warp; the 12 corner-plane passes into a
//     per-warp force buffer in the same slot map run as 8 groups separated by __syncwarp only (each pass
//     is injective over the lanes, passes of different z parity never meet; the first group stores the
//     64 owned nodes, the others read-modify-write); then a node phase (4 nodes per lane) stores the 27
//     tile-interior nodes and adds the others with one red.global.add.v4.f32 each.
// ---------------------------------------------------------------------------------------------
constexpr int WZ_W = 4;  // independent warps per CTA
struct WzWarp {
    alignas(16) f4 uh[2][132];
    alignas(16) f4 F[132];
    alignas(16) float mh[2][64];
};
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ldg_stream(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ldg_stream1(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
// node-phase node n (0..124) -> halo node (X, Y, Z): n < 80: Z = n / 16, X = n % 16 / 4, Y = n % 4 (a
// quarter-warp covers X in {2j, 2j+1} x Y = 0..3, so 4X + Y is distinct mod 8); then the X = 4 / Y = 4
// faces, 9 per plane Z
__device__ __forceinline__ void wz_node(int n, int &X, int &Y, int &Z) {
    if (n < 80) { Z = n >> 4; X = (n >> 2) & 3; Y = n & 3; }
    else { const int m = n - 80, j = m % 9; Z = m / 9; X = j < 5 ? 4 : j - 5; Y = j < 5 ? j : 4; }
}
// role: local id | neighbour slot << 6 | owned << 9 | interior << 10 | u-halo slot (5X + 26Y + Z) << 11;
// -1 = none
__device__ __forceinline__ int wz_role(int n) {
    if (n >= 125) return -1;
    int X, Y, Z;
    wz_node(n, X, Y, Z);
    const int dp = ((X >> 2) << 2) | ((Y >> 2) << 1) | (Z >> 2);
    const int interior = (X >= 1 && X <= 3 && Y >= 1 && Y <= 3 && Z >= 1 && Z <= 3);
    return local_id(X & 3, Y & 3, Z & 3) | (dp << 6) | ((dp == 0) << 9) | (interior << 10) | ((5 * X + 26 * Y + Z) << 11);
}

// packed upper-triangle element e -> row r (kofs(r) <= e < kofs(r + 1)) and column
__host__ __device__ constexpr int krow(int e) {
    int r = 0;
    while (r < 8 && kofs(r + 1) <= e) r++;
    return r;
}
__host__ __device__ constexpr int kcol(int e) { return krow(e) + (e - kofs(krow(e))); }

// compressed-tangent apply for the two cells of a lane at once (KC): every value a float2 (cell A, cell B),
// so each operation is one paired fp32 instruction (FFMA2 / FMUL2 / FADD2 on sm_100).  k holds the 24
// interleaved pairs (A_e, B_e) of q_U = (x, y, z) (3; w = sqrt(1 - x^2 - y^2 - z^2) >= 1/2), W = S V (9,
// row-major), c psi_ij (6), c (a, b) x 3 pairs (6); d = dG (raw nodal sums);
// P = c U (C : (U^T dG W)) W^T = c (C_F : (dG S)) S with C in the SVD frame (S symmetric, so V^T S = W^T;
// DESIGN §4).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ void quat_rot2(float2 w, float2 x, float2 y, float2 z, float2 R[9]) {
    const float2 two = f2(2.f, 2.f), one = f2(1.f, 1.f);
    const float2 xx = mul2(x, x), yy = mul2(y, y), zz = mul2(z, z);
    const float2 xy = mul2(x, y), xz = mul2(x, z), yz = mul2(y, z), wx = mul2(w, x), wy = mul2(w, y), wz = mul2(w, z);
    R[0] = sub2(one, mul2(two, add2(yy, zz)));
    R[1] = mul2(two, sub2(xy, wz));
    R[2] = mul2(two, add2(xz, wy));
    R[3] = mul2(two, add2(xy, wz));
    R[4] = sub2(one, mul2(two, add2(xx, zz)));
    R[5] = mul2(two, sub2(yz, wx));
    R[6] = mul2(two, sub2(xz, wy));
    R[7] = mul2(two, add2(yz, wx));
    R[8] = sub2(one, mul2(two, add2(xx, yy)));
}
constexpr int KC_CHUNKS = KC_REALS / 2;  // 12 chunks of (A_e, B_e, A_e+1, B_e+1) per pair slot
__device__ __forceinline__ void kc_apply2(const float *k, const float2 d[9], float2 P[9]) {
    auto el = [&](int e) { return f2(k[4 * (e >> 1) + 2 * (e & 1)], k[4 * (e >> 1) + 2 * (e & 1) + 1]); };
    float2 RU[9];
    {
        const float2 x = el(0), y = el(1), z = el(2);
        const float2 s = fma2(x, x, fma2(y, y, mul2(z, z)));
        const float2 t = sub2(f2(1.f, 1.f), s);  // = w^2 >= 1/4 (an absent partner: 1)
        const float2 w = mul2(t, f2(rsqrtf(t.x), rsqrtf(t.y)));
        quat_rot2(w, x, y, z, RU);
    }
    float2 T1[9], Xh[9];  // Xh = RU^T dG W
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            float2 v = mul2(RU[i], d[j]);
            v = fma2(RU[3 + i], d[3 + j], v);
            T1[3 * i + j] = fma2(RU[6 + i], d[6 + j], v);
        }
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            float2 v = mul2(T1[3 * i], el(3 + j));
            v = fma2(T1[3 * i + 1], el(6 + j), v);
            Xh[3 * i + j] = fma2(T1[3 * i + 2], el(9 + j), v);
        }
    float2 Yh[9];
    const float2 D00 = el(12), D11 = el(13), D22 = el(14), D01 = el(15), D12 = el(16), D02 = el(17);
    Yh[0] = fma2(D00, Xh[0], fma2(D01, Xh[4], mul2(D02, Xh[8])));
    Yh[4] = fma2(D01, Xh[0], fma2(D11, Xh[4], mul2(D12, Xh[8])));
    Yh[8] = fma2(D02, Xh[0], fma2(D12, Xh[4], mul2(D22, Xh[8])));
    {
        const float2 a = el(18), b = el(19);  // pair (0, 1)
        Yh[1] = fma2(a, Xh[1], mul2(b, Xh[3]));
        Yh[3] = fma2(b, Xh[1], mul2(a, Xh[3]));
    }
    {
        const float2 a = el(20), b = el(21);  // pair (0, 2)
        Yh[2] = fma2(a, Xh[2], mul2(b, Xh[6]));
        Yh[6] = fma2(b, Xh[2], mul2(a, Xh[6]));
    }
    {
        const float2 a = el(22), b = el(23);  // pair (1, 2)
        Yh[5] = fma2(a, Xh[5], mul2(b, Xh[7]));
        Yh[7] = fma2(b, Xh[5], mul2(a, Xh[7]));
    }
    float2 T2[9];  // P = RU Yh W^T
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            float2 v = mul2(RU[3 * i], Yh[j]);
            v = fma2(RU[3 * i + 1], Yh[3 + j], v);
            T2[3 * i + j] = fma2(RU[3 * i + 2], Yh[6 + j], v);
        }
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            float2 v = mul2(T2[3 * i], el(3 + 3 * j));
            v = fma2(T2[3 * i + 1], el(4 + 3 * j), v);
            P[3 * i + j] = fma2(T2[3 * i + 2], el(5 + 3 * j), v);
        }
}

template <bool KC, int MINB = 3, bool LIST = false, bool GR = false>
__global__ void __launch_bounds__(32 * WZ_W, MINB)
    k_hvp_wz(int T_, const int *__restrict__ nplus, const unsigned long long *__restrict__ cmask,
             const int *__restrict__ hascells, const float *__restrict__ K, const int *__restrict__ kstart,
             const float *__restrict__ nmass, const f4 *__restrict__ u, f4 *__restrict__ Hu, double *__restrict__ uHu,
             const CGSlot *__restrict__ cgs, int cgj, double cgthr, const DevScalars *__restrict__ sc,
             const int *__restrict__ tlist, int ntl, const int *__restrict__ jdev) {
    // items: tiles 0..T_-1, or the listed tiles tlist[0..ntl) (slab ranks: the interface tiles first, so
    // their halo exchange overlaps the interior tiles' launch).  jdev (graph-captured PCG): the
    // iteration index, its p.Hp slot and the threshold come from device memory
    const int N = LIST ? ntl : T_;
    __shared__ WzWarp SW[WZ_W];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WzWarp &S = SW[wid];
    // programmatic dependent launch: everything up to the first tile's tangent and metadata reads data the
    // previous kernel does not write (the tangent, tile tables), so it runs before griddepcontrol.wait and
    // overlaps the previous kernel's tail; u, the CG scalars and the iteration index are read after it.
    // In a captured graph (GR, jdev) the wait comes first: with the prologue ahead of it the replayed
    // iteration counts broke (the index read raced with the previous node's write); the
    // 45-number form (!KC) also waits first (its 90 prefetched tangent registers spilled ahead of the wait)
    constexpr bool EARLY = KC && !GR;
    pdl_trigger();
    if (!EARLY) pdl_wait();
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    const int zp = lane >> 4, lx = (lane >> 2) & 3, ly = lane & 3;
    const int lA = lx * 16 + ly * 4 + 2 * zp;  // cell A's local position (B = lA + 1)
    const int hb = 5 * lx + 26 * ly + 2 * zp;  // u-halo slot of cell A's (0,0,0) corner
    int role[4];
#pragma unroll
    for (int r = 0; r < 4; r++) role[r] = wz_role(lane + 32 * r);
    for (int i = lane; i < 132; i += 32) S.F[i] = mk4<float>(0.f, 0.f, 0.f, 0.f);
    const uint64_t pol = l2_evict_first_policy();
    const int G = gridDim.x * WZ_W, t0 = blockIdx.x * WZ_W + wid;
    // tile metadata, spread over lanes 0-11: neighbours (lane 0 = the tile itself), kstart, has, cmask
    // halves; one 32-bit load per lane at a per-lane base + stride t, no use until the next iteration
    const int *mbase = lane < 8 ? nplus + lane : lane == 8 ? kstart : lane == 9 ? hascells
                                                                      : reinterpret_cast<const int *>(cmask) + (lane - 10);
    const int mstride = lane < 8 ? 8 : lane < 10 ? 1 : 2;
    auto load_meta = [&](int i) -> int {  // metadata of item i's tile
        if (i >= N || lane >= 12) return 0;
        const int t = LIST ? __ldg(tlist + i) : i;
        return lane == 0 ? t : __ldg(mbase + (int64_t)mstride * t);
    };
    struct TileK {
        int has, pA, pB;         // the tile has cells; this lane's cells A / B are present
        unsigned sb;             // chunk stride in bytes (16 n)
        int e44, d44;            // element 44 of cell A at ka + e44, of cell B at kbp + e44 - 3 d44
        const float *ka, *kbp;   // this lane's first chunk of cell A / B
    };
    auto tile_k = [&](int t, int meta) -> TileK {
        TileK q;
        q.has = __shfl_sync(FULL, meta, 9);
        const int ks = __shfl_sync(FULL, meta, 8);
        const unsigned clo = (unsigned)__shfl_sync(FULL, meta, 10), chi = (unsigned)__shfl_sync(FULL, meta, 11);
        if (t >= N) q.has = 0;
        const unsigned word = lA < 32 ? clo : chi;
        q.pA = q.has ? (int)((word >> (lA & 31)) & 1u) : 0;
        q.pB = q.has ? (int)((word >> ((lA + 1) & 31)) & 1u) : 0;
        if (KC) {  // compressed: one pair slot per lane holding a cell, KC_CHUNKS interleaved chunks
            const unsigned pm = __ballot_sync(FULL, q.pA | q.pB);
            q.sb = 16u * (unsigned)__popc(pm);
            q.ka = K + ks + 4 * __popc(pm & lt);
            q.kbp = q.ka;
            q.e44 = q.d44 = 0;
            return q;
        }
        const unsigned pmA = __ballot_sync(FULL, q.pA), pmB = __ballot_sync(FULL, q.pB);
        const int nA = __popc(pmA), n = nA + __popc(pmB);
        const int sA = __popc(pmA & lt), sB = nA + __popc(pmB & lt);
        q.sb = 16u * (unsigned)n;
        q.ka = K + ks + 4 * sA;
        q.kbp = K + ks + 4 * sB;
        q.e44 = 44 * n + sA - 4 * sA;  // element 44 of slot s at 44 n + s, relative to ka / kbp
        q.d44 = sB - sA;
        return q;
    };
    float k[90];
    // chunk c < 11 of slot s at 4 (c n + s), element 44 at 44 n + s (k_off): chunk c at (byte)
    // ka + c * 16 n, one IMAD.WIDE per load.  Chunk c of cell X (off 0 = A, 45 = B) -> k
    auto kload = [&](const TileK &q, int off, int c) {
        if (KC) {  // off 0: chunks 0..6, off 45: chunks 7..11 (the 12 calls per cell map onto 12 chunks)
            const int cc = (off ? 7 : 0) + c;
            if (c >= 7 || cc >= KC_CHUNKS || !(q.pA | q.pB)) return;
            const float4 v = ldg_stream(reinterpret_cast<const float *>(reinterpret_cast<const char *>(q.ka) +
                                                                        (uint64_t)q.sb * (uint64_t)cc), pol);
            k[4 * cc] = v.x; k[4 * cc + 1] = v.y; k[4 * cc + 2] = v.z; k[4 * cc + 3] = v.w;
            return;
        }
        if (!(off ? q.pB : q.pA)) return;
        const float *p = off ? q.kbp : q.ka;
        if (c < 11) {
            const float4 v = ldg_stream(reinterpret_cast<const float *>(reinterpret_cast<const char *>(p) +
                                                                        (uint64_t)q.sb * (uint64_t)c), pol);
            k[off + 4 * c] = v.x; k[off + 4 * c + 1] = v.y; k[off + 4 * c + 2] = v.z; k[off + 4 * c + 3] = v.w;
        } else {
            k[off + 44] = ldg_stream1(p + q.e44 - (off ? 3 * q.d44 : 0), pol);
        }
    };
    // shared addresses: this warp's halo / mass buffers (buffer b at + b UHB / + b MHB) and force buffer
    const uint32_t s_uh = smem_u32(&S.uh[0][0]), s_mh = smem_u32(&S.mh[0][0]), s_F = smem_u32(&S.F[0]);
    constexpr uint32_t UHB = 132 * 16, MHB = 64 * 4;
    // tile t: u halo + owned masses -> shared buffer b (cp.async, one group).  Node-phase nodes
    // n = lane + 32 r: r < 2 are the tile's own 64 nodes (X, Y, Z < 4: owned, the tile itself), r >= 2 the
    // 61 face nodes of neighbour tiles
    auto halo = [&](int t, int b, int meta) {
        const int has = __shfl_sync(FULL, meta, 9), ts = __shfl_sync(FULL, meta, 0);
        int tt[4];
#pragma unroll
        for (int r = 2; r < 4; r++) tt[r] = __shfl_sync(FULL, meta, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
        if (t < N) {
            const uint32_t bu = s_uh + (uint32_t)b * UHB, bm = s_mh + (uint32_t)b * MHB;
            const f4 *ut = u + (int64_t)ts * 64;
            const float *mt = nmass + (int64_t)ts * 64;
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const int loc = role[r] & 63, h = role[r] >> 11;
                cp_async16s(bu + 16u * h, ut + loc);
                cp_async4s(bm + 4u * loc, mt + loc);
            }
#pragma unroll
            for (int r = 2; r < 4; r++) {
                if (role[r] < 0) continue;
                const int loc = role[r] & 63, h = role[r] >> 11;
                if (has && tt[r] >= 0) cp_async16s(bu + 16u * h, u + ((int64_t)tt[r] * 64 + loc));
                else sts4z(bu + 16u * h);
            }
        }
        cp_async_commit();
    };
    int mcur = load_meta(t0);
    int mnext = load_meta(t0 + G);
    TileK cur = tile_k(t0, mcur);
#pragma unroll
    for (int c = 0; c < 12; c++) { kload(cur, 0, c); kload(cur, 45, c); }
    if (EARLY) pdl_wait();
    if (GR) {
        cgj = *jdev;
        uHu = const_cast<double *>(cgs[cgj].pHp);
        cgthr = sc->cg_thr;
    }
    if (cgs != nullptr) {  // inside PCG: nothing to do once converged / stopped at negative curvature
        const double rr = warp_sum(cgs[cgj].rr[lane]);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    halo(t0, 0, mcur);
    double acc = 0.0;
    int it = 0;
    for (int t = t0; t < N; t += G, it++) {  // t: item index
        const int b = it & 1;
        const int mnn = load_meta(t + 2 * G);
        const TileK nxt = tile_k(t + G, mnext);
        cp_async_wait<0>();
        __syncwarp();
        const f4 *uh = S.uh[b];
        float2 P2[9];  // (cell A, cell B) pairs
        if (cur.has) {
            // ---- dG of cells A and B from the 12 nodes (ox, oy) x z-plane q = 0, 1, 2
            float Dx[3][3], Dy[3][3], Sz[3][3];  // [plane][component]
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const f4 w00 = uh[hb + q], w01 = uh[hb + 26 + q], w10 = uh[hb + 5 + q], w11 = uh[hb + 31 + q];
                const float a00[3] = {w00.x, w00.y, w00.z}, a01[3] = {w01.x, w01.y, w01.z};
                const float a10[3] = {w10.x, w10.y, w10.z}, a11[3] = {w11.x, w11.y, w11.z};
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const float s1 = a11[a] - a00[a], s2 = a10[a] - a01[a];
                    Dx[q][a] = s1 + s2;  // sum over oy of (x=1) - (x=0)
                    Dy[q][a] = s1 - s2;  // sum over ox of (y=1) - (y=0)
                    Sz[q][a] = (a00[a] + a11[a]) + (a01[a] + a10[a]);
                }
            }
            float dA[9], dB[9];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                dA[3 * a] = Dx[0][a] + Dx[1][a]; dA[3 * a + 1] = Dy[0][a] + Dy[1][a]; dA[3 * a + 2] = Sz[1][a] - Sz[0][a];
                dB[3 * a] = Dx[1][a] + Dx[2][a]; dB[3 * a + 1] = Dy[1][a] + Dy[2][a]; dB[3 * a + 2] = Sz[2][a] - Sz[1][a];
            }
            float2 d2[9];
#pragma unroll
            for (int r = 0; r < 9; r++) d2[r] = make_float2(dA[r], dB[r]);
            if (KC) {
                kc_apply2(k, d2, P2);
            } else {
            float PA[9], PB[9];
            // ---- P = K dG (symmetric, packed upper triangle), element by element
#pragma unroll
            for (int r = 0; r < 9; r++) { PA[r] = 0.f; PB[r] = 0.f; }
#pragma unroll
            for (int e = 0; e < 45; e++) {
                const int r = krow(e), c = kcol(e);
                PA[r] += k[e] * dA[c];
                if (c != r) PA[c] += k[e] * dA[r];
            }
#pragma unroll
            for (int e = 0; e < 45; e++) {
                const int r = krow(e), c = kcol(e);
                PB[r] += k[45 + e] * dB[c];
                if (c != r) PB[c] += k[45 + e] * dB[r];
            }
#pragma unroll
            for (int r = 0; r < 9; r++) P2[r] = make_float2(PA[r], PB[r]);
            }
            float2 q2 = f2(0.f, 0.f);
#pragma unroll
            for (int r = 0; r < 9; r++) {
                P2[r].x = cur.pA ? P2[r].x : 0.f;  // absent cells: k holds stale numbers
                P2[r].y = cur.pB ? P2[r].y : 0.f;
                q2 = fma2(P2[r], d2[r], q2);
            }
            acc += (double)(q2.x + q2.y);
        }
        // k is free: start the next tile's loads; they overlap the scatter and the node phase (issuing the
        // second half after the scatter measured slower: 87.3 vs 86.2 us at cfg4)
#pragma unroll
        for (int c = 0; c < 12; c++) { kload(nxt, 0, c); kload(nxt, 45, c); }
        halo(t + G, b ^ 1, mnext);
        // corner force of cell X at (sx, sy, sz) = +-(Px +- Py) +- Pz per component: 4 sums g; the value
        // of corner (ox, oy, oz): (sx, sy) = (+,+) -> g0/g1, (-,-) -> -g1/-g0, (+,-) -> g2/g3,
        // (-,+) -> -g3/-g2 (first for sz = +1, second for sz = -1)
        auto corner = [&](const float g[4], int ox, int oy, int oz) -> float {
            if (ox && oy) return oz ? g[0] : g[1];
            if (!ox && !oy) return oz ? -g[1] : -g[0];
            if (ox) return oz ? g[2] : g[3];
            return oz ? -g[3] : -g[2];
        };
        if (cur.has) {
            float gA[3][4], gB[3][4];
#pragma unroll
            for (int a = 0; a < 3; a++) {  // both cells at once (paired adds)
                const float2 e1 = add2(P2[3 * a], P2[3 * a + 1]), e2 = sub2(P2[3 * a], P2[3 * a + 1]), z = P2[3 * a + 2];
                const float2 g0 = add2(e1, z), g1 = sub2(e1, z), g2 = add2(e2, z), g3 = sub2(e2, z);
                gA[a][0] = g0.x; gA[a][1] = g1.x; gA[a][2] = g2.x; gA[a][3] = g3.x;
                gB[a][0] = g0.y; gB[a][1] = g1.y; gB[a][2] = g2.y; gB[a][3] = g3.y;
            }
            auto cf = [&](int ox, int oy, int q) -> f4 {  // this lane's force on node (ox, oy, plane q)
                f4 f;
                f.w = 0.f;
                if (q == 0) {
                    f.x = corner(gA[0], ox, oy, 0); f.y = corner(gA[1], ox, oy, 0); f.z = corner(gA[2], ox, oy, 0);
                } else if (q == 2) {
                    f.x = corner(gB[0], ox, oy, 1); f.y = corner(gB[1], ox, oy, 1); f.z = corner(gB[2], ox, oy, 1);
                } else {
                    f.x = corner(gA[0], ox, oy, 1) + corner(gB[0], ox, oy, 0);
                    f.y = corner(gA[1], ox, oy, 1) + corner(gB[1], ox, oy, 0);
                    f.z = corner(gA[2], ox, oy, 1) + corner(gB[2], ox, oy, 0);
                }
                return f;
            };
            {
                // 8 groups: node z = 2 zp + q, so passes of different q parity never meet the same node; a
                // group pairs an even-q pass with an odd-q pass (two independent read-modify-writes), and
                // the first group (ox, oy) = (0, 0), q = 0, 1 covers the 64 nodes x, y, z < 4 exactly once:
                // plain stores (those nodes are not zeroed by the node phase)
#ifdef MPL_DEBUG
                // race check of the __syncwarp-only scatter (debug build): every force-buffer slot written in
                // a group is claimed once in a per-warp bitmap; a second claim in the same group traps
                __shared__ unsigned dbg_claim[WZ_W][5];
                auto claim = [&](int slot) {
                    const unsigned bit = 1u << (slot & 31), old = atomicOr(&dbg_claim[wid][slot >> 5], bit);
                    DASSERT(slot >= 0 && slot < 132 && !(old & bit));
                };
                auto release = [&]() {
                    __syncwarp();
                    if (lane < 5) dbg_claim[wid][lane] = 0u;
                    __syncwarp();
                };
                release();
#define MPL_CLAIM(s) claim(s)
#define MPL_RELEASE() release()
#else
#define MPL_CLAIM(s) \
    do {             \
    } while (0)
#define MPL_RELEASE() \
    do {              \
    } while (0)
#endif
                {
                    const f4 f0 = cf(0, 0, 0), f1 = cf(0, 0, 1);
                    MPL_CLAIM(hb);
                    MPL_CLAIM(hb + 1);
                    S.F[hb] = f0;
                    S.F[hb + 1] = f1;
                    __syncwarp();
                    MPL_RELEASE();
                }
#pragma unroll
                for (int g = 0; g < 7; g++) {
                    // even passes after (0,0,0): (0,0,2) (0,1,0) (0,1,2) (1,0,0) (1,0,2) (1,1,0) (1,1,2);
                    // odd passes (0,1,1) (1,0,1) (1,1,1) with the first three groups that start a new (ox, oy)
                    const int e = g + 1, eox = e >> 2, eoy = (e >> 1) & 1, eq = (e & 1) * 2;
                    f4 *fe = &S.F[hb + 5 * eox + 26 * eoy + eq];
                    const f4 fe_ = cf(eox, eoy, eq);
                    MPL_CLAIM(hb + 5 * eox + 26 * eoy + eq);
                    if ((g & 1) == 1) {  // g = 1, 3, 5: odd pass (ox, oy) = e's
                        MPL_CLAIM(hb + 5 * eox + 26 * eoy + 1);
                        f4 *fo = &S.F[hb + 5 * eox + 26 * eoy + 1];
                        const f4 fo_ = cf(eox, eoy, 1);
                        const f4 a = *fe, b = *fo;
                        *fe = mk4<float>(a.x + fe_.x, a.y + fe_.y, a.z + fe_.z, 0.f);
                        *fo = mk4<float>(b.x + fo_.x, b.y + fo_.y, b.z + fo_.z, 0.f);
                    } else {
                        const f4 a = *fe;
                        *fe = mk4<float>(a.x + fe_.x, a.y + fe_.y, a.z + fe_.z, 0.f);
                    }
                    __syncwarp();
                    MPL_RELEASE();
                }
#undef MPL_CLAIM
#undef MPL_RELEASE
            }
        }
        // ---- node phase: forces + lumped mass term, stored (interior) or added atomically (faces)
        {
            const uint32_t bu = s_uh + (uint32_t)b * UHB, bm = s_mh + (uint32_t)b * MHB;
            const int ts = __shfl_sync(FULL, mcur, 0);
            f4 *Ht = Hu + (int64_t)ts * 64;
            float am = 0.f;  // sum of m |u|^2 over this lane's owned nodes
#pragma unroll
            for (int r = 0; r < 2; r++) {  // the tile's own nodes: scatter stored them; plus m_i u_i
                const int loc = role[r] & 63, h = role[r] >> 11;
                f4 f = mk4<float>(0.f, 0.f, 0.f, 0.f);
                if (cur.has) f = lds4(s_F + 16u * h);
                const float mm = lds1(bm + 4u * loc);
                const f4 w = lds4(bu + 16u * h);
                f.x = fmaf(mm, w.x, f.x); f.y = fmaf(mm, w.y, f.y); f.z = fmaf(mm, w.z, f.z);
                am = fmaf(mm, fmaf(w.x, w.x, fmaf(w.y, w.y, w.z * w.z)), am);
                if ((role[r] >> 10) & 1) Ht[loc] = mk4<float>(f.x, f.y, f.z, 0.f);
                else if (f.x != 0.f || f.y != 0.f || f.z != 0.f) atomic_add3<float>(Ht + loc, f.x, f.y, f.z);
            }
            acc += (double)am;
            if (cur.has) {
                int tt[4];
#pragma unroll
                for (int r = 2; r < 4; r++) tt[r] = __shfl_sync(FULL, mcur, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
#pragma unroll
                for (int r = 2; r < 4; r++) {  // face nodes of the neighbour tiles: added atomically
                    if (role[r] < 0) continue;
                    const int loc = role[r] & 63, h = role[r] >> 11;
                    const f4 f = lds4(s_F + 16u * h);
                    sts4z(s_F + 16u * h);
                    if (tt[r] >= 0 && (f.x != 0.f || f.y != 0.f || f.z != 0.f))
                        atomic_add3<float>(Hu + ((int64_t)tt[r] * 64 + loc), f.x, f.y, f.z);
                }
            }
        }
        __syncwarp();  // node phase done reading uh[b] / mh[b] before they are refilled
        mcur = mnext;
        mnext = mnn;
        cur = nxt;
    }
    cp_async_wait<0>();
    if (uHu) {
        const double v = warp_sum(acc);
        if (lane == 0 && v != 0.0) atomicAdd(&uHu[(blockIdx.x * WZ_W + wid) % NSTRIPE], v);
    }
}

// ---------------------------------------------------------------------------------------------
// v7 (MPL_HVP_KERNEL=wh): one warp per HALF tile, one cell per lane.  The wz kernel holds both cells'
// tangents (90 registers) to keep a whole tile of loads in flight, which caps it at 12 warps / SM
// where it is latency bound; here a lane holds one cell's 45 numbers, so 20 warps / SM fit.
//   * item i = 2 t + h (h = the half: cells lx in {2h, 2h+1}); persistent warps strided by an even
//     count, so a warp always works on the same half h and its node roles are fixed;
//   * lane = 16 (lx - 2h) + 4 ly + lz, i.e. local cell l = 32 h + lane: in the tile's natural compact
//     order (layout 3: slot = rank of l among the tile's cells) a warp's slots are contiguous;
//   * the half's 3 x 5 x 5 node halo at shared slot 25 x + 5 y + 2 z (every quarter-warp's 16-byte
//     accesses conflict-free), 8 scatter passes into a per-warp force buffer, then 3 nodes per lane:
//     the 9 nodes all of whose cells lie in the half are stored, the others (incl. the x = 2 plane
//     shared with the other half) added atomically; the lumped-mass term of an owned node is added by
//     the half whose cells own its x (x in {2h, 2h+1}).
// ---------------------------------------------------------------------------------------------
constexpr int WH_W = 4;  // warps per CTA
template <class T> struct WhWarp {
    alignas(16) vec4<T> uh[2][80];
    alignas(16) vec4<T> F[80];
    alignas(16) T mh[2][32];
};
__device__ __forceinline__ double2 ldg_stream2d(const double *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ldg_stream1d(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// chunk c (16 bytes) of a tangent slot and the remainder element 44, both precisions
template <class T> __device__ __forceinline__ void wh_chunk(const T *p, uint64_t pol, T *k);
template <> __device__ __forceinline__ void wh_chunk<float>(const float *p, uint64_t pol, float *k) {
    const float4 v = ldg_stream(p, pol);
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
}
template <> __device__ __forceinline__ void wh_chunk<double>(const double *p, uint64_t pol, double *k) {
    const double2 v = ldg_stream2d(p, pol);
    k[0] = v.x; k[1] = v.y;
}
__device__ __forceinline__ float wh_one(const float *p, uint64_t pol) { return ldg_stream1(p, pol); }
__device__ __forceinline__ double wh_one(const double *p, uint64_t pol) { return ldg_stream1d(p, pol); }
// role of halo node n (0..74) of half h: local id | neighbour slot << 6 | mass << 9 | interior << 10 |
// shared slot << 11 | mass index << 18; -1 = none
__device__ __forceinline__ int wh_role(int n, int h) {
    if (n >= 75) return -1;
    const int x = n / 25, Y = (n / 5) % 5, Z = n % 5, X = 2 * h + x;
    const int dp = ((X >> 2) << 2) | ((Y >> 2) << 1) | (Z >> 2);
    const int mass = (x < 2 && Y < 4 && Z < 4);
    const int interior = (x == 1 && Y >= 1 && Y <= 3 && Z >= 1 && Z <= 3);
    const int midx = mass ? x * 16 + Y * 4 + Z : 0;
    return local_id(X & 3, Y & 3, Z & 3) | (dp << 6) | (mass << 9) | (interior << 10) | ((25 * x + 5 * Y + 2 * Z) << 11) |
           (midx << 18);
}

template <class T, int MINB>
__global__ void __launch_bounds__(32 * WH_W, MINB)
    k_hvp_wh(int T_, const int *__restrict__ nplus, const unsigned long long *__restrict__ cmask,
             const int *__restrict__ hascells, const T *__restrict__ K, const int *__restrict__ kstart,
             const T *__restrict__ nmass, const vec4<T> *__restrict__ u, vec4<T> *__restrict__ Hu,
             double *__restrict__ uHu, const CGSlot *__restrict__ cgs, int cgj, double cgthr,
             const DevScalars *__restrict__ sc) {
    using V4 = vec4<T>;
    constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
    __shared__ WhWarp<T> SW[WH_W];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WhWarp<T> &S = SW[wid];
    pdl_trigger();
    pdl_wait();
    if (cgs != nullptr) {
        const double rr = warp_sum(cgs[cgj].rr[lane]);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    const int G = gridDim.x * WH_W, i0 = blockIdx.x * WH_W + wid;  // G even: item parity fixed
    const int h = i0 & 1;
    const int lx = 2 * h + (lane >> 4), ly = (lane >> 2) & 3, lz = lane & 3;
    const int hb = 25 * (lx - 2 * h) + 5 * ly + 2 * lz;  // shared slot of the cell's (0,0,0) corner
    int role[3];
#pragma unroll
    for (int r = 0; r < 3; r++) role[r] = wh_role(lane + 32 * r, h);
    for (int i = lane; i < 80; i += 32) S.F[i] = mk4<T>(T(0), T(0), T(0), T(0));
    const uint64_t pol = l2_evict_first_policy();
    const int NI = 2 * T_;
    const int *mbase = lane < 8 ? nplus + lane : lane == 8 ? kstart : lane == 9 ? hascells
                                                                      : reinterpret_cast<const int *>(cmask) + (lane - 10);
    const int mstride = lane < 8 ? 8 : lane < 10 ? 1 : 2;
    auto load_meta = [&](int it_) -> int {  // metadata of item it_'s tile, spread over lanes 0-11
        if (it_ >= NI || lane >= 12) return 0;
        const int t = it_ >> 1;
        return lane == 0 ? t : __ldg(mbase + (int64_t)mstride * t);
    };
    struct TileK {
        int has, pres;
        unsigned sb;  // chunk stride in bytes (16 n)
        int e44;      // element 44 at ka + e44
        const T *ka;
    };
    auto tile_k = [&](int it_, int meta) -> TileK {
        TileK q;
        q.has = __shfl_sync(FULL, meta, 9);
        const int ks = __shfl_sync(FULL, meta, 8);
        const unsigned clo = (unsigned)__shfl_sync(FULL, meta, 10), chi = (unsigned)__shfl_sync(FULL, meta, 11);
        if (it_ >= NI) q.has = 0;
        const unsigned word = h ? chi : clo;
        q.pres = q.has ? (int)((word >> lane) & 1u) : 0;
        const int n = __popc(clo) + __popc(chi);
        const int sl = (h ? __popc(clo) : 0) + __popc(word & lt);
        q.sb = 16u * (unsigned)n;
        q.ka = K + ks + VEC * sl;
        q.e44 = 44 * n + sl - VEC * sl;
        return q;
    };
    T k[45];
    auto kload_all = [&](const TileK &q) {
        if (!q.pres) return;
#pragma unroll
        for (int c = 0; c < NCH; c++)
            wh_chunk<T>(reinterpret_cast<const T *>(reinterpret_cast<const char *>(q.ka) + (uint64_t)q.sb * (uint64_t)c),
                        pol, k + VEC * c);
        k[44] = wh_one(q.ka + q.e44, pol);
    };
    auto halo = [&](int it_, int b, int meta) {
        const int has = __shfl_sync(FULL, meta, 9);
        int tt[3];
#pragma unroll
        for (int r = 0; r < 3; r++) tt[r] = __shfl_sync(FULL, meta, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
        if (it_ < NI) {
#pragma unroll
            for (int r = 0; r < 3; r++) {
                if (role[r] < 0) continue;
                const int loc = role[r] & 63, mass = (role[r] >> 9) & 1, hs = (role[r] >> 11) & 127,
                          mi = role[r] >> 18;
                if ((has || mass) && tt[r] >= 0) {
                    const int64_t nd = (int64_t)tt[r] * 64 + loc;
#pragma unroll
                    for (int qq = 0; qq < (int)(sizeof(V4) / 16); qq++)
                        cp_async16(reinterpret_cast<char *>(&S.uh[b][hs]) + 16 * qq,
                                   reinterpret_cast<const char *>(u + nd) + 16 * qq);
                    if (mass) cp_async_real<T>(&S.mh[b][mi], nmass + nd);
                } else {
                    S.uh[b][hs] = mk4<T>(T(0), T(0), T(0), T(0));
                    if (mass) S.mh[b][mi] = T(0);
                }
            }
        }
        cp_async_commit();
    };
    int mcur = load_meta(i0);
    int mnext = load_meta(i0 + G);
    TileK cur = tile_k(i0, mcur);
    kload_all(cur);
    halo(i0, 0, mcur);
    double acc = 0.0;
    int itc = 0;
    for (int it_ = i0; it_ < NI; it_ += G, itc++) {
        const int b = itc & 1;
        const int mnn = load_meta(it_ + 2 * G);
        const TileK nxt = tile_k(it_ + G, mnext);
        cp_async_wait<0>();
        __syncwarp();
        const V4 *uh = S.uh[b];
        T P[9];
        if (cur.has) {
            T dG[9];
            {
                T Dx[2][3], Dy[2][3], Sz[2][3];
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    const V4 w00 = uh[hb + q * 2], w01 = uh[hb + 5 + q * 2], w10 = uh[hb + 25 + q * 2],
                             w11 = uh[hb + 30 + q * 2];
                    const T a00[3] = {w00.x, w00.y, w00.z}, a01[3] = {w01.x, w01.y, w01.z};
                    const T a10[3] = {w10.x, w10.y, w10.z}, a11[3] = {w11.x, w11.y, w11.z};
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        const T s1 = a11[a] - a00[a], s2 = a10[a] - a01[a];
                        Dx[q][a] = s1 + s2;
                        Dy[q][a] = s1 - s2;
                        Sz[q][a] = (a00[a] + a11[a]) + (a01[a] + a10[a]);
                    }
                }
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    dG[3 * a] = Dx[0][a] + Dx[1][a];
                    dG[3 * a + 1] = Dy[0][a] + Dy[1][a];
                    dG[3 * a + 2] = Sz[1][a] - Sz[0][a];
                }
            }
#pragma unroll
            for (int r = 0; r < 9; r++) P[r] = T(0);
#pragma unroll
            for (int e = 0; e < 45; e++) {
                const int r = krow(e), c = kcol(e);
                P[r] += k[e] * dG[c];
                if (c != r) P[c] += k[e] * dG[r];
            }
            T qf = T(0);
#pragma unroll
            for (int r = 0; r < 9; r++) {
                P[r] = cur.pres ? P[r] : T(0);
                qf += P[r] * dG[r];
            }
            acc += (double)qf;
        }
        kload_all(nxt);
        halo(it_ + G, b ^ 1, mnext);
        if (cur.has) {
            T g4[3][4];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                const T e1 = P[3 * a] + P[3 * a + 1], e2 = P[3 * a] - P[3 * a + 1], z = P[3 * a + 2];
                g4[a][0] = e1 + z; g4[a][1] = e1 - z; g4[a][2] = e2 + z; g4[a][3] = e2 - z;
            }
            auto corner = [&](const T g[4], int ox, int oy, int oz) -> T {
                if (ox && oy) return oz ? g[0] : g[1];
                if (!ox && !oy) return oz ? -g[1] : -g[0];
                if (ox) return oz ? g[2] : g[3];
                return oz ? -g[3] : -g[2];
            };
#pragma unroll
            for (int ox = 0; ox < 2; ox++)
#pragma unroll
                for (int oy = 0; oy < 2; oy++)
#pragma unroll
                    for (int oz = 0; oz < 2; oz++) {
                        V4 *fp = &S.F[hb + 25 * ox + 5 * oy + 2 * oz];
                        const V4 o = *fp;
                        *fp = mk4<T>(o.x + corner(g4[0], ox, oy, oz), o.y + corner(g4[1], ox, oy, oz),
                                     o.z + corner(g4[2], ox, oy, oz), T(0));
                        __syncwarp();
                    }
        }
        int tt[3];
#pragma unroll
        for (int r = 0; r < 3; r++) tt[r] = __shfl_sync(FULL, mcur, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
#pragma unroll
        for (int r = 0; r < 3; r++) {
            if (role[r] < 0) continue;
            const int loc = role[r] & 63, mass = (role[r] >> 9) & 1, interior = (role[r] >> 10) & 1,
                      hs = (role[r] >> 11) & 127, mi = role[r] >> 18;
            V4 f = mk4<T>(T(0), T(0), T(0), T(0));
            if (cur.has) {
                f = S.F[hs];
                S.F[hs] = mk4<T>(T(0), T(0), T(0), T(0));
            }
            if (!(cur.has || mass) || tt[r] < 0) continue;
            if (mass) {
                const T mm = S.mh[b][mi];
                if (mm > T(0)) {
                    const V4 w = uh[hs];
                    f.x += mm * w.x; f.y += mm * w.y; f.z += mm * w.z;
                    acc += (double)(mm * (w.x * w.x + w.y * w.y + w.z * w.z));
                }
            }
            const int64_t nd = (int64_t)tt[r] * 64 + loc;
            if (interior) Hu[nd] = mk4<T>(f.x, f.y, f.z, T(0));
            else if (f.x != T(0) || f.y != T(0) || f.z != T(0)) atomic_add3<T>(Hu + nd, f.x, f.y, f.z);
        }
        __syncwarp();
        mcur = mnext;
        mnext = mnn;
        cur = nxt;
    }
    cp_async_wait<0>();
    if (uHu) {
        const double v = warp_sum(acc);
        if (lane == 0 && v != 0.0) atomicAdd(&uHu[(blockIdx.x * WH_W + wid) % NSTRIPE], v);
    }
}

int g_num_sms = 0;

template <bool KC, int MINB, bool LIST, bool GR = false>
mpl_status launch_wz(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                     double cgthr, const int *tlist, int ntl, const int *jdev = nullptr) {
    static int per_sm = 0;
    if (per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_wz<KC, MINB, LIST, GR>, 32 * WZ_W, 0));
        per_sm = occ > 0 ? occ : 1;
    }
    // persistent: one wave of (SMs x resident CTAs), tiles strided by the global warp count
    int grid = g_num_sms * per_sm;
    const int need = ((tlist ? ntl : ctx->T) + WZ_W - 1) / WZ_W;
    if (grid > need) grid = need;
    if (grid < 1) return MPL_OK;
    MPL_CUDA(launch_pdl(k_hvp_wz<KC, MINB, LIST, GR>, grid, 32 * WZ_W, 0, ctx->stream, ctx->T, (const int *)ctx->t_nplus.p,
                        (const unsigned long long *)ctx->t_cmask.p, (const int *)ctx->t_hascells.p,
                        (const float *)ctx->K.p, (const int *)(KC ? ctx->t_kstart2.p : ctx->t_kstart.p),
                        (const float *)owned_mass(ctx),
                        (const f4 *)u_tile, (f4 *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p,
                        tlist, ntl, jdev));
    ctx->launches++;
    return MPL_OK;
}

template <class T, int MINB>
mpl_status launch_wh(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                     double cgthr) {
    static int per_sm = 0;
    if (per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_wh<T, MINB>, 32 * WH_W, 0));
        per_sm = occ > 0 ? occ : 1;
    }
    int grid = g_num_sms * per_sm;
    const int need = (2 * ctx->T + WH_W - 1) / WH_W;
    if (grid > need) grid = need;
    MPL_CUDA(launch_pdl(k_hvp_wh<T, MINB>, grid, 32 * WH_W, 0, ctx->stream, ctx->T, (const int *)ctx->t_nplus.p,
                        (const unsigned long long *)ctx->t_cmask.p, (const int *)ctx->t_hascells.p,
                        (const T *)ctx->K.p, (const int *)ctx->t_kstart.p, (const T *)owned_mass(ctx),
                        (const vec4<T> *)u_tile, (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr,
                        (const DevScalars *)ctx->scalars.p));
    ctx->launches++;
    return MPL_OK;
}

}  // namespace

// fp32 HVP kernel (MPL_HVP_KERNEL): "wz" (default, k_hvp_wz) or "wh" (k_hvp_wh<float, 5>, the half-tile
// reference kernel); fp64 always runs k_hvp_wh<double, 3>.
int hvp_variant() {
    static int variant = -1;
    if (variant < 0) {
        const char *e = getenv("MPL_HVP_KERNEL");
        variant = (e && e[0] == 'w' && e[1] == 'h') ? 1 : 0;
    }
    return variant;
}
bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("MPL_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// Tangent slot order k_linearize writes (k_off): 1 = compact kz order (k_hvp_wz), 3 = natural compact
// order, slot = rank of the cell in its tile (k_hvp_wh, fp64 and MPL_HVP_KERNEL=wh).
int hvp_kz_layout(int precision) {
    if (precision != 32 || hvp_variant() == 1) return 3;
    return 1;
}

// Hu (tile-dense) must be zero on every node that receives atomics (all non-interior nodes).
template <class T>
mpl_status launch_hvp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                      double cgthr, const int *tlist, int ntl, const int *jdev) {
    if (ctx->T == 0) return MPL_OK;
    if (jdev) {  // graph-captured PCG: fp32 compressed-tangent k_hvp_wz only
        if (sizeof(T) == 8 || hvp_variant() == 1 || !ctx->kc_now || tlist) return MPL_ERR_UNSUPPORTED;
        return launch_wz<true, 3, false, true>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, nullptr, 0, jdev);
    }
    if (tlist && (sizeof(T) == 8 || hvp_variant() == 1)) return MPL_ERR_UNSUPPORTED;  // tile lists: k_hvp_wz only
    if (sizeof(T) == 8) return launch_wh<T, 3>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);  // 45 doubles per lane
    if (hvp_variant() == 1) return launch_wh<T, 5>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (ctx->kc_now) {  // compressed tangent; MPL_KC_MINB: CTAs per SM requested from ptxas (2, the default:
                        // ptxas takes 168 registers, 3 CTAs of 4 warps still fit, cfg4 68.9 us isolated / 75.4
                        // in the solve; 3: 148 registers, 70.2 / 76.5; 4: 128 + 8 B spilled, 16 warps, 73.0 /
                        // 77.4; 5: 96 registers + 192 B spilled, 117 us)
        static int minb = -1;
        if (minb < 0) {
            const char *e = getenv("MPL_KC_MINB");
            minb = e ? atoi(e) : 2;
        }
        if (tlist) return launch_wz<true, 3, true>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, tlist, ntl);
        if (minb == 3) return launch_wz<true, 3, false>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, nullptr, 0);
        if (minb == 2) return launch_wz<true, 2, false>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, nullptr, 0);
        return launch_wz<true, 4, false>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, nullptr, 0);
    }
    if (tlist) return launch_wz<false, 3, true>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, tlist, ntl);
    return launch_wz<false, 3, false>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr, nullptr, 0);
}

template mpl_status launch_hvp<float>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double,
                                      const int *, int, const int *);
template mpl_status launch_hvp<double>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double,
                                       const int *, int, const int *);
