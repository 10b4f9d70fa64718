// k_hvp.cu — SURVEY §8(a) row a6, the graded kernel: the matrix-free Hessian-vector product
//     (H u)_i = m_i u_i + sum_{c ∋ i} (K_c : dG_c(u)) grad w_ic ,   dG_c(u) = sum_j u_j (x) grad w_jc
// (App. B: H = M + d^2 E/dv^2; grad w_ic = (x_i - x_c)/(2 dx^2); "matrix-free
// PCG" P:495), with K_c the cached 9x9 symmetric tangent of the quadrature point (k_linearize).
//
// Persistent CTAs (64 threads, one tile of 4^3 cells at a time, tiles strided by gridDim):
//   * tangent blocks (<= 64 cells x 180 B) stream through an NS-stage shared-memory ring filled by
//     cp.async.bulk (TMA bulk copy, SASS UBLKCP) completing on an mbarrier, issued NS-1 tiles ahead;
//   * the 5^3 node halo of u is prefetched with 16-byte cp.async (LDGSTS) into the same stage;
//   * P = K dG (81 FMA), scattered to the 8 corners in 8 barrier-separated passes (pass o adds to
//     node cell+o, injective, so shared adds never collide);
//   * the 27 nodes whose 8 cells all lie in the tile are stored, the face nodes get one float4 atomic.
// u . Hu = sum_i m_i |u_i|^2 + sum_c dG:K:dG is accumulated exactly (striped fp64 accumulators).
#include <cstdlib>

#include "mpl_common.cuh"

namespace {

constexpr int HVP_THREADS = 64;
constexpr int HVP_STAGES = 3;

__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

__device__ __forceinline__ int64_t halo_node(int t, const int *__restrict__ nplus, int h) {
    int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
    int dp = ((hx >> 2) << 2) | ((hy >> 2) << 1) | (hz >> 2);
    int tt = dp ? nplus[8 * t + dp] : t;
    if (tt < 0) return -1;
    return (int64_t)tt * 64 + local_id(hx & 3, hy & 3, hz & 3);
}

template <class T> __device__ __forceinline__ void atomic_add3(vec4<T> *p, T x, T y, T z);
template <> __device__ __forceinline__ void atomic_add3<float>(f4 *p, float x, float y, float z) {
    atomicAdd(reinterpret_cast<float4 *>(p), make_float4(x, y, z, 0.f));
}
template <> __device__ __forceinline__ void atomic_add3<double>(d4 *p, double x, double y, double z) {
    atomicAdd(&p->x, x);
    atomicAdd(&p->y, y);
    atomicAdd(&p->z, z);
}

// ---- PTX wrappers: mbarrier + bulk copy (TMA) + cp.async -------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class T> __device__ __forceinline__ void lds_vec(const T *p, T *k);
template <> __device__ __forceinline__ void lds_vec<float>(const float *p, float *k) {
    float4 v = *reinterpret_cast<const float4 *>(p);
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
}
template <> __device__ __forceinline__ void lds_vec<double>(const double *p, double *k) {
    double2 v = *reinterpret_cast<const double2 *>(p);
    k[0] = v.x; k[1] = v.y;
}

template <class T> struct HvpSmem {
    alignas(128) T K[HVP_STAGES][64 * 45];
    alignas(16) vec4<T> uh[HVP_STAGES][125];
    T F[3][128];
    uint64_t bar[HVP_STAGES];
    int has[HVP_STAGES], cs[HVP_STAGES], ncp[HVP_STAGES];
    double red[2];
    int stop;
};

template <class T>
__device__ __forceinline__ void hvp_issue(HvpSmem<T> &S, int stage, int t, int T_, const int *__restrict__ nplus,
                                          const int *__restrict__ cstart, const int *__restrict__ hascells,
                                          const T *__restrict__ K, const vec4<T> *__restrict__ u) {
    const int tid = threadIdx.x;
    if (t < T_) {
        const int cs = cstart[t], ncp = cstart[t + 1] - cs, has = hascells[t];
        if (tid == 0) {
            S.has[stage] = has;
            S.cs[stage] = cs;
            S.ncp[stage] = ncp;
            const uint32_t bytes = (uint32_t)(ncp * 45 * sizeof(T));
            mbar_expect_tx(&S.bar[stage], bytes);
            if (bytes) bulk_g2s(S.K[stage], K + (int64_t)cs * 45, bytes, &S.bar[stage]);
        }
        for (int h = tid; h < 125; h += HVP_THREADS) {
            int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
            bool owned = hx < 4 && hy < 4 && hz < 4;
            int64_t n = (has || owned) ? halo_node(t, nplus, h) : -1;
            if (n >= 0) {
#pragma unroll
                for (int q = 0; q < (int)(sizeof(vec4<T>) / 16); q++)
                    cp_async16(reinterpret_cast<char *>(&S.uh[stage][h]) + 16 * q,
                               reinterpret_cast<const char *>(u + n) + 16 * q);
            } else {
                S.uh[stage][h] = mk4<T>(0, 0, 0, 0);
            }
        }
    }
    cp_async_commit();
}

template <class T>
__global__ void __launch_bounds__(HVP_THREADS) k_hvp_tma(int T_, const int *__restrict__ nplus,
                                                         const int *__restrict__ cstart,
                                                         const uint8_t *__restrict__ clocal,
                                                         const int *__restrict__ hascells, const T *__restrict__ K,
                                                         const T *__restrict__ nmass, const vec4<T> *__restrict__ u,
                                                         vec4<T> *__restrict__ Hu, double *__restrict__ uHu,
                                                         const CGSlot *__restrict__ cgs, int cgj, double cgthr,
                                                         const DevScalars *__restrict__ sc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    HvpSmem<T> &S = *reinterpret_cast<HvpSmem<T> *>(smem_raw);
    const int tid = threadIdx.x;
    if (cgs != nullptr) {  // inside PCG: skip once converged / broken down (uniform per CTA)
        double rr = stripe_sum_bcast(cgs[cgj].rr);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    if (tid == 0) {
        for (int s = 0; s < HVP_STAGES; s++) mbar_init(&S.bar[s], 1);
        mbar_fence_init();
    }
    for (int i = tid; i < 3 * 128; i += HVP_THREADS) (&S.F[0][0])[i] = T(0);
    __syncthreads();
    const int G = gridDim.x;
    const int t0 = blockIdx.x;
    // prologue: tiles it = 0 .. NS-2
#pragma unroll
    for (int s = 0; s < HVP_STAGES - 1; s++) hvp_issue<T>(S, s, t0 + s * G, T_, nplus, cstart, hascells, K, u);
    double acc = 0.0;
    int it = 0;
    for (int t = t0; t < T_; t += G, it++) {
        const int stage = it % HVP_STAGES;
        // refill the stage freed at the end of the previous iteration (NS-1 tiles ahead)
        hvp_issue<T>(S, (it + HVP_STAGES - 1) % HVP_STAGES, t + (HVP_STAGES - 1) * G, T_, nplus, cstart, hascells, K, u);
        cp_async_wait<HVP_STAGES - 1>();
        mbar_wait(&S.bar[stage], (uint32_t)((it / HVP_STAGES) & 1));
        __syncthreads();
        const int has = S.has[stage], cs = S.cs[stage], ncp = S.ncp[stage];
        const vec4<T> *uh = S.uh[stage];
        // ---- cell phase ----------------------------------------------------------------------
        int l = 0xFF;
        if (tid < ncp) l = clocal[cs + tid];
        const bool act = (l != 0xFF);
        const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
        T P[9];
        if (act) {
            constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
            const T *Ks = S.K[stage];
            T k[45];
#pragma unroll
            for (int c = 0; c < NCH; c++) lds_vec<T>(Ks + (c * ncp + tid) * VEC, k + c * VEC);
            k[44] = Ks[NCH * VEC * ncp + tid];
            T dG[9];
#pragma unroll
            for (int a = 0; a < 9; a++) dG[a] = T(0);
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                vec4<T> w = uh[((lx + ox) * 5 + ly + oy) * 5 + lz + oz];
                const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                dG[0] += w.x * s0; dG[1] += w.x * s1; dG[2] += w.x * s2;
                dG[3] += w.y * s0; dG[4] += w.y * s1; dG[5] += w.y * s2;
                dG[6] += w.z * s0; dG[7] += w.z * s1; dG[8] += w.z * s2;
            }
#pragma unroll
            for (int r = 0; r < 9; r++) P[r] = k[kidx(r, r)] * dG[r];
#pragma unroll
            for (int r = 0; r < 9; r++)
#pragma unroll
                for (int q = r + 1; q < 9; q++) {
                    P[r] += k[kidx(r, q)] * dG[q];
                    P[q] += k[kidx(r, q)] * dG[r];
                }
            T qf = T(0);
#pragma unroll
            for (int r = 0; r < 9; r++) qf += P[r] * dG[r];
            acc += (double)qf;
        }
        if (has) {
#pragma unroll
            for (int o = 0; o < 8; o++) {
                if (act) {
                    const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                    const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                    const int h = ((lx + ox) * 5 + ly + oy) * 5 + lz + oz;
                    S.F[0][h] += P[0] * s0 + P[1] * s1 + P[2] * s2;
                    S.F[1][h] += P[3] * s0 + P[4] * s1 + P[5] * s2;
                    S.F[2][h] += P[6] * s0 + P[7] * s1 + P[8] * s2;
                }
                __syncthreads();
            }
        }
        // ---- node phase: store interior nodes, atomically add face nodes ----------------------
        for (int h = tid; h < 125; h += HVP_THREADS) {
            int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
            bool owned = hx < 4 && hy < 4 && hz < 4;
            T f0 = S.F[0][h], f1 = S.F[1][h], f2 = S.F[2][h];
            S.F[0][h] = S.F[1][h] = S.F[2][h] = T(0);
            if (!has && !owned) continue;
            bool interior = hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3;
            int64_t n = halo_node(t, nplus, h);
            if (n < 0) continue;
            if (owned) {
                T m = nmass[n];
                if (m > T(0)) {
                    vec4<T> w = uh[h];
                    f0 += m * w.x; f1 += m * w.y; f2 += m * w.z;
                    acc += (double)(m * (w.x * w.x + w.y * w.y + w.z * w.z));
                }
            }
            if (interior) Hu[n] = mk4<T>(f0, f1, f2, T(0));
            else if (f0 != T(0) || f1 != T(0) || f2 != T(0)) atomic_add3<T>(Hu + n, f0, f1, f2);
        }
        __syncthreads();  // stage and F free for reuse
    }
    cp_async_wait<0>();
    if (uHu) {
        double v = warp_sum(acc);
        if ((tid & 31) == 0) S.red[tid >> 5] = v;
        __syncthreads();
        if (tid == 0) {
            double s = S.red[0] + S.red[1];
            if (s != 0.0) atomicAdd(&uHu[blockIdx.x % NSTRIPE], s);
        }
    }
}

// v2 (default): one tile per 64-thread CTA, tangent loaded straight into registers with 16-byte
// loads coalesced across the tile's cells; ~14 CTAs resident per SM hide the latency.
template <class T> __device__ __forceinline__ void ldg_vec(const T *p, T *k);
template <> __device__ __forceinline__ void ldg_vec<float>(const float *p, float *k) {
    float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
}
template <> __device__ __forceinline__ void ldg_vec<double>(const double *p, double *k) {
    double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    k[0] = v.x; k[1] = v.y;
}

template <class T>
__global__ void __launch_bounds__(64) k_hvp_reg(const int *__restrict__ nplus, const int *__restrict__ cstart,
                                                const uint8_t *__restrict__ clocal, const int *__restrict__ hascells,
                                                const T *__restrict__ K, const T *__restrict__ nmass,
                                                const vec4<T> *__restrict__ u, vec4<T> *__restrict__ Hu,
                                                double *__restrict__ uHu, const CGSlot *__restrict__ cgs, int cgj,
                                                double cgthr, const DevScalars *__restrict__ sc) {
    __shared__ vec4<T> uh[125];
    __shared__ T Fs[3][128];
    __shared__ double red[2];
    const int t = blockIdx.x, tid = threadIdx.x;
    if (cgs != nullptr) {
        double rr = stripe_sum_bcast(cgs[cgj].rr);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    const int has = hascells[t];
    const int cs = cstart[t], ncp = cstart[t + 1] - cs;
    constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
    T k[45];
    int l = 0xFF;
    if (tid < ncp) {
        l = clocal[cs + tid];
        const T *base = K + (int64_t)cs * 45;
#pragma unroll
        for (int c = 0; c < NCH; c++) ldg_vec<T>(base + ((int64_t)c * ncp + tid) * VEC, k + c * VEC);
        k[44] = __ldg(base + (int64_t)NCH * VEC * ncp + tid);
    }
    for (int h = tid; h < 125; h += 64) {
        int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        bool owned = hx < 4 && hy < 4 && hz < 4;
        int64_t n = (has || owned) ? halo_node(t, nplus, h) : -1;
        uh[h] = n >= 0 ? u[n] : mk4<T>(0, 0, 0, 0);
        Fs[0][h] = Fs[1][h] = Fs[2][h] = T(0);
    }
    __syncthreads();
    double acc = 0.0;
    const bool act = (l != 0xFF);
    const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    T P[9];
    if (act) {
        T dG[9];
#pragma unroll
        for (int a = 0; a < 9; a++) dG[a] = T(0);
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            vec4<T> w = uh[((lx + ox) * 5 + ly + oy) * 5 + lz + oz];
            const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
            dG[0] += w.x * s0; dG[1] += w.x * s1; dG[2] += w.x * s2;
            dG[3] += w.y * s0; dG[4] += w.y * s1; dG[5] += w.y * s2;
            dG[6] += w.z * s0; dG[7] += w.z * s1; dG[8] += w.z * s2;
        }
#pragma unroll
        for (int r = 0; r < 9; r++) P[r] = k[kidx(r, r)] * dG[r];
#pragma unroll
        for (int r = 0; r < 9; r++)
#pragma unroll
            for (int q = r + 1; q < 9; q++) {
                P[r] += k[kidx(r, q)] * dG[q];
                P[q] += k[kidx(r, q)] * dG[r];
            }
        T qf = T(0);
#pragma unroll
        for (int r = 0; r < 9; r++) qf += P[r] * dG[r];
        acc += (double)qf;
    }
    if (has) {
#pragma unroll
        for (int o = 0; o < 8; o++) {
            if (act) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                const int h = ((lx + ox) * 5 + ly + oy) * 5 + lz + oz;
                Fs[0][h] += P[0] * s0 + P[1] * s1 + P[2] * s2;
                Fs[1][h] += P[3] * s0 + P[4] * s1 + P[5] * s2;
                Fs[2][h] += P[6] * s0 + P[7] * s1 + P[8] * s2;
            }
            __syncthreads();
        }
    }
    for (int h = tid; h < 125; h += 64) {
        int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        bool owned = hx < 4 && hy < 4 && hz < 4;
        if (!has && !owned) continue;
        bool interior = hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3;
        int64_t n = halo_node(t, nplus, h);
        if (n < 0) continue;
        T f0 = Fs[0][h], f1 = Fs[1][h], f2 = Fs[2][h];
        if (owned) {
            T m = nmass[n];
            if (m > T(0)) {
                vec4<T> w = uh[h];
                f0 += m * w.x; f1 += m * w.y; f2 += m * w.z;
                acc += (double)(m * (w.x * w.x + w.y * w.y + w.z * w.z));
            }
        }
        if (interior) Hu[n] = mk4<T>(f0, f1, f2, T(0));
        else if (f0 != T(0) || f1 != T(0) || f2 != T(0)) atomic_add3<T>(Hu + n, f0, f1, f2);
    }
    if (uHu) {
        double v = warp_sum(acc);
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        if (tid == 0) {
            double s = red[0] + red[1];
            if (s != 0.0) atomicAdd(&uHu[blockIdx.x % NSTRIPE], s);
        }
    }
}

int g_num_sms = 0;

}  // namespace

// Hu (tile-dense) must be zero on every node that receives atomics (all non-interior nodes).
template <class T>
mpl_status launch_hvp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                      double cgthr) {
    if (ctx->T == 0) return MPL_OK;
    static int variant = -1;
    if (variant < 0) {
        const char *e = getenv("MPL_HVP_KERNEL");
        variant = (e && e[0] == 't') ? 1 : 0;  // "tma" = persistent bulk-copy ring, default = register v2
    }
    if (variant == 0) {
        k_hvp_reg<T><<<ctx->T, 64, 0, ctx->stream>>>(
            (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
            (const int *)ctx->t_hascells.p, (const T *)ctx->K.p, (const T *)ctx->n_mass.p, (const vec4<T> *)u_tile,
            (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
        ctx->launches++;
        MPL_CUDA(cudaGetLastError());
        return MPL_OK;
    }
    static bool attr_set[2] = {false, false};
    const size_t smem = sizeof(HvpSmem<T>);
    const int pi = sizeof(T) == 8;
    if (!attr_set[pi]) {
        MPL_CUDA(cudaFuncSetAttribute(k_hvp_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set[pi] = true;
    }
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hvp_tma<T>, HVP_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    int grid = g_num_sms * per_sm;
    if (grid > ctx->T) grid = ctx->T;
    k_hvp_tma<T><<<grid, HVP_THREADS, smem, ctx->stream>>>(
        ctx->T, (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
        (const int *)ctx->t_hascells.p, (const T *)ctx->K.p, (const T *)ctx->n_mass.p, (const vec4<T> *)u_tile,
        (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
    ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

template mpl_status launch_hvp<float>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double);
template mpl_status launch_hvp<double>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double);
