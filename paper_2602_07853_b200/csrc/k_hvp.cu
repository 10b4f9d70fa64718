// k_hvp.cu — SURVEY §8(a) row a6, the graded kernel: the matrix-free Hessian-vector product
//     (H u)_i = m_i u_i + sum_{c ∋ i} (K_c : dG_c(u)) grad w_ic ,   dG_c(u) = sum_j u_j (x) grad w_jc
// (App. B: H = M + d^2 E/dv^2; grad w_ic = (x_i - x_c)/(2 dx^2); "matrix-free
// PCG" P:495), with K_c the cached 9x9 symmetric tangent of the quadrature point (k_linearize).
//
// Default kernel k_hvp_pipe: persistent CTAs (64 threads, one tile of 4^3 cells at a time, tiles
// strided by gridDim):
//   * tangent blocks (<= 64 cells x 180 B) stream through an NS-stage shared-memory ring filled by
//     cp.async.bulk (TMA bulk copy, SASS UBLKCP) completing on an mbarrier, NS tiles in flight;
//   * the 5^3 node halo of u, the owned masses and the cell ids are prefetched with cp.async (LDGSTS)
//     into the same stage;
//   * P = K dG (81 FMA), scattered to the 8 corners in 8 passes into a per-warp force buffer (pass o
//     adds to node cell+o, injective over the warp, so only __syncwarp separates passes);
//   * the 27 nodes whose 8 cells all lie in the tile are stored, the face nodes get one float4 atomic.
// Two block barriers per tile.  u . Hu = sum_i m_i |u_i|^2 + sum_c dG:K:dG is accumulated exactly
// (striped fp64 accumulators).
#include <cstdlib>

#include "mpl_common.cuh"

namespace {


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

// v2 (MPL_HVP_KERNEL=reg): one tile per 64-thread CTA, tangent loaded straight into registers with
// 16-byte loads coalesced across the tile's cells; ~14 CTAs resident per SM hide the latency.
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
                                                const T *__restrict__ K, const int *__restrict__ kstart,
                                                const int *__restrict__ ncell, const T *__restrict__ nmass,
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
    const int cs = cstart[t], n = ncell[t];
    constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
    T k[45];
    int l = 0xFF;
    const int cj = hvp_cell(tid), ks = hvp_slot(tid, n);
    if (has && cj < n) {  // tiles outside the slab (ghost planes) carry no tangent
        l = clocal[cs + cj];
        const T *base = K + kstart[t];
#pragma unroll
        for (int c = 0; c < NCH; c++) ldg_vec<T>(base + ((int64_t)c * n + ks) * VEC, k + c * VEC);
        k[44] = __ldg(base + (int64_t)NCH * VEC * n + ks);
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

// ---------------------------------------------------------------------------------------------
// v3 (default): persistent, software-pipelined.  One 64-thread CTA walks tiles t0, t0+G, ... with
// an NS-stage shared-memory ring: the tile's contiguous tangent block arrives by one cp.async.bulk
// (TMA bulk copy, SASS UBLKCP) completing on an mbarrier; the 5^3 u halo, the 64 owned masses and
// the 64 local cell ids arrive by cp.async, all issued NS-1 tiles ahead.  Each thread owns two halo
// roles (h = tid, tid + 64) whose coordinates / neighbour slot / interior flag are computed once per
// launch, so the per-tile integer work of v2 (h/25, h/5, table lookups) disappears; the neighbour
// table and tile metadata of the tile after next are prefetched into registers one iteration early.
// ---------------------------------------------------------------------------------------------
template <class T, int NS> struct PipeSmem {
    alignas(128) T K[NS][64 * 45];
    alignas(16) vec4<T> uh[NS][128];
    alignas(16) T mh[NS][64];
    alignas(16) uint8_t cl[NS][64];
    T F[2][3][128];  // per-warp corner-force accumulators
    uint64_t bar[NS];
    int nb[NS + 1][8];    // metadata ring is one deeper than the data ring: the slot written for tile
    int meta[NS + 1][4];  // it+NS is never a slot of a tile still in flight or being consumed
    double red[2];
};

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <class T> __device__ __forceinline__ void cp_async_real(T *dst, const T *src);
template <> __device__ __forceinline__ void cp_async_real<float>(float *dst, const float *src) { cp_async4(dst, src); }
template <> __device__ __forceinline__ void cp_async_real<double>(double *dst, const double *src) { cp_async8(dst, src); }

// halo role: bits 0-5 local node id in its tile, 6-8 neighbour slot dp, 9 owned (dp == 0),
// 10 interior (all 8 cells in this tile), 11-17 halo index h; -1 = no role
__device__ __forceinline__ int make_role(int h) {
    if (h >= 125) return -1;
    const int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
    const int dp = ((hx >> 2) << 2) | ((hy >> 2) << 1) | (hz >> 2);
    const int loc = local_id(hx & 3, hy & 3, hz & 3);
    const int interior = (hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3);
    return loc | (dp << 6) | ((dp == 0) << 9) | (interior << 10) | (h << 11);
}

template <class T, int NS>
__global__ void __launch_bounds__(64) k_hvp_pipe(int T_, const int *__restrict__ nplus, const int *__restrict__ cstart,
                                                 const uint8_t *__restrict__ clocal, const int *__restrict__ hascells,
                                                 const T *__restrict__ K, const int *__restrict__ kstart,
                                                const int *__restrict__ ncell, const T *__restrict__ nmass,
                                                 const vec4<T> *__restrict__ u, vec4<T> *__restrict__ Hu,
                                                 double *__restrict__ uHu, const CGSlot *__restrict__ cgs, int cgj,
                                                 double cgthr, const DevScalars *__restrict__ sc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeSmem<T, NS> &S = *reinterpret_cast<PipeSmem<T, NS> *>(smem_raw);
    const int tid = threadIdx.x;
    if (cgs != nullptr) {  // inside PCG: skip once converged / broken down (uniform per CTA)
        double rr = stripe_sum_bcast(cgs[cgj].rr);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    const int role0 = make_role(tid), role1 = make_role(tid + 64);
    if (tid == 0) {
        for (int s = 0; s < NS; s++) mbar_init(&S.bar[s], 1);
        mbar_fence_init();
    }
    for (int i = tid; i < 2 * 3 * 128; i += 64) (&S.F[0][0][0])[i] = T(0);
    const int G = gridDim.x, t0 = blockIdx.x;
    // register-staged metadata of the next tile to issue: tid < 8 neighbour slot tid, 8 cs, 9 ce, 10 has
    auto load_meta = [&](int t) -> int {
        if (t >= T_) return 0;
        if (tid < 8) return tid ? nplus[8 * t + tid] : t;
        if (tid == 8) return cstart[t];
        if (tid == 9) return ncell[t];
        if (tid == 10) return hascells[t];
        if (tid == 11) return kstart[t];
        return 0;
    };
    auto put_meta = [&](int s, int t, int reg) {
        if (tid < 8) S.nb[s][tid] = reg;
        if (tid >= 8 && tid < 12) S.meta[s][tid - 8] = reg;  // cs, n (real cells), has, kstart
        (void)t;
    };
    auto issue_role = [&](int s, int mi, int has, int role) {
        if (role < 0) return;
        const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1, h = role >> 11;
        const int tt = S.nb[mi][dp];
        if ((has || owned) && tt >= 0) {
            const int64_t n = (int64_t)tt * 64 + loc;
#pragma unroll
            for (int q = 0; q < (int)(sizeof(vec4<T>) / 16); q++)
                cp_async16(reinterpret_cast<char *>(&S.uh[s][h]) + 16 * q, reinterpret_cast<const char *>(u + n) + 16 * q);
            if (owned) cp_async_real<T>(&S.mh[s][loc], nmass + n);
        } else {
            S.uh[s][h] = mk4<T>(0, 0, 0, 0);
            if (owned) S.mh[s][loc] = T(0);
        }
    };
    // all threads: after a barrier that published S.nb[s] / S.meta[s]
    auto issue = [&](int s, int mi, int t) {
        if (t < T_) {
            const int cs = S.meta[mi][0], n = S.meta[mi][1], has = S.meta[mi][2], kb = S.meta[mi][3];
            const int nk = has ? n : 0;
            if (tid == 0) {
                const uint32_t bytes = (uint32_t)(((45 * nk + 3) & ~3) * sizeof(T));  // t_kcnt: multiple of 16 B
                mbar_expect_tx(&S.bar[s], bytes);
                if (bytes) bulk_g2s(S.K[s], K + kb, bytes, &S.bar[s]);
            }
            if (tid * 4 < nk) cp_async4(&S.cl[s][tid * 4], clocal + cs + tid * 4);
            issue_role(s, mi, has, role0);
            issue_role(s, mi, has, role1);
        }
        cp_async_commit();
    };
    __syncthreads();
    // prologue: tiles 0 .. NS-1 of this CTA in flight
    for (int s = 0; s < NS; s++) {
        const int t = t0 + s * G;
        put_meta(s, t, load_meta(t));
        __syncthreads();
        issue(s, s, t);
    }
    int reg = load_meta(t0 + NS * G);
    double acc = 0.0;
    int it = 0;
    for (int t = t0; t < T_; t += G, it++) {
        const int st = it % NS;
        const int mc = it % (NS + 1), mn = (it + NS) % (NS + 1);
        cp_async_wait<NS - 1>();
        mbar_wait(&S.bar[st], (uint32_t)((it / NS) & 1));
        __syncthreads();  // (B) stage st complete for every thread
        const int ncp = S.meta[mc][1], has = S.meta[mc][2];  // ncp: real cells of the tile
        const vec4<T> *uh = S.uh[st];
        // ---- cell phase: P = K dG, corner forces added to per-warp F ---------------------------
        const int cj = hvp_cell(tid), ks = hvp_slot(tid, ncp);
        const int l = (has && cj < ncp) ? (int)S.cl[st][cj] : 0xFF;
        if (l != 0xFF) {
            const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
            constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
            const T *Ks = S.K[st];
            T k[45];
#pragma unroll
            for (int c = 0; c < NCH; c++) lds_vec<T>(Ks + (c * ncp + ks) * VEC, k + c * VEC);
            k[44] = Ks[NCH * VEC * ncp + ks];
            T dG[9];
#pragma unroll
            for (int a = 0; a < 9; a++) dG[a] = T(0);
            const int hb = (lx * 5 + ly) * 5 + lz;
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                vec4<T> w = uh[hb + ox * 25 + oy * 5 + oz];
                const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                dG[0] += w.x * s0; dG[1] += w.x * s1; dG[2] += w.x * s2;
                dG[3] += w.y * s0; dG[4] += w.y * s1; dG[5] += w.y * s2;
                dG[6] += w.z * s0; dG[7] += w.z * s1; dG[8] += w.z * s2;
            }
            T P[9];
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
            // pass o adds to node cell + o: injective over the warp's cells, so no lane conflicts;
            // each warp has its own F, so passes need only __syncwarp (no block barrier)
            T *Fw = S.F[tid >> 5][0];
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                const int h = hb + ox * 25 + oy * 5 + oz;
                Fw[h] += P[0] * s0 + P[1] * s1 + P[2] * s2;
                Fw[128 + h] += P[3] * s0 + P[4] * s1 + P[5] * s2;
                Fw[256 + h] += P[6] * s0 + P[7] * s1 + P[8] * s2;
                __syncwarp(__activemask());
            }
        }
        // node-phase inputs that live in the stage go to registers, so the stage can be refilled
        // right after the barrier
        int64_t nidx[2];
        T fm[2][3];
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            nidx[r] = -1;
            fm[r][0] = fm[r][1] = fm[r][2] = T(0);
            if (role < 0) continue;
            const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1, h = role >> 11;
            if (!has && !owned) continue;
            const int tt = dp ? S.nb[mc][dp] : t;
            if (tt < 0) continue;
            nidx[r] = (int64_t)tt * 64 + loc;
            if (owned) {
                const T m = S.mh[st][loc];
                if (m > T(0)) {
                    const vec4<T> w = uh[h];
                    fm[r][0] = m * w.x; fm[r][1] = m * w.y; fm[r][2] = m * w.z;
                    acc += (double)(m * (w.x * w.x + w.y * w.y + w.z * w.z));
                }
            }
        }
        put_meta(mn, t + NS * G, reg);
        __syncthreads();  // (C) F complete; stage st consumed; metadata of tile t + NS G visible
        issue(st, mn, t + NS * G);
        reg = load_meta(t + (NS + 1) * G);
        // ---- node phase (two fixed roles per thread) -------------------------------------------
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            if (role < 0) continue;
            const int h = role >> 11, interior = (role >> 10) & 1;
            const T f0 = S.F[0][0][h] + S.F[1][0][h] + fm[r][0], f1 = S.F[0][1][h] + S.F[1][1][h] + fm[r][1],
                    f2 = S.F[0][2][h] + S.F[1][2][h] + fm[r][2];
            S.F[0][0][h] = S.F[0][1][h] = S.F[0][2][h] = S.F[1][0][h] = S.F[1][1][h] = S.F[1][2][h] = T(0);
            if (nidx[r] < 0) continue;
            if (interior) Hu[nidx[r]] = mk4<T>(f0, f1, f2, T(0));
            else if (f0 != T(0) || f1 != T(0) || f2 != T(0)) atomic_add3<T>(Hu + nidx[r], f0, f1, f2);
        }
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

// ---------------------------------------------------------------------------------------------
// v4 (MPL_HVP_KERNEL=rp): persistent, register-pipelined.  The next tile's tangent goes straight
// from HBM into the registers that just finished the current tile's K dG (16-byte loads coalesced
// across the tile's cells, issued before the scatter / node phase, so those phases and the other
// resident CTAs cover the load latency); the u halo / masses / cell ids of the next tile are
// cp.async'ed into the other half of a 2-slot shared buffer.  No tangent staging in shared memory:
// ~8 KB of shared memory per CTA, so registers alone bound occupancy.
// ---------------------------------------------------------------------------------------------
template <class T> struct RpSmem {
    alignas(16) vec4<T> uh[2][128];
    alignas(16) T mh[2][64];
    alignas(16) uint8_t cl[2][64];
    T F[2][3][128];
    int nb[3][8];
    int meta[3][4];  // cs, n (real cells), has, kstart
    double red[2];
};

template <class T, int MINB>
__global__ void __launch_bounds__(64, MINB) k_hvp_rp(int T_, const int *__restrict__ nplus, const int *__restrict__ cstart,
                                               const uint8_t *__restrict__ clocal, const int *__restrict__ hascells,
                                               const T *__restrict__ K, const int *__restrict__ kstart,
                                                const int *__restrict__ ncell, const T *__restrict__ nmass,
                                               const vec4<T> *__restrict__ u, vec4<T> *__restrict__ Hu,
                                               double *__restrict__ uHu, const CGSlot *__restrict__ cgs, int cgj,
                                               double cgthr, const DevScalars *__restrict__ sc) {
    __shared__ RpSmem<T> S;
    const int tid = threadIdx.x;
    if (cgs != nullptr) {
        double rr = stripe_sum_bcast(cgs[cgj].rr);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
    const int role0 = make_role(tid), role1 = make_role(tid + 64);
    for (int i = tid; i < 2 * 3 * 128; i += 64) (&S.F[0][0][0])[i] = T(0);
    const int G = gridDim.x, t0 = blockIdx.x;
    auto load_meta = [&](int t) -> int {
        if (t >= T_) return 0;
        if (tid < 8) return tid ? nplus[8 * t + tid] : t;
        if (tid == 8) return cstart[t];
        if (tid == 9) return ncell[t];
        if (tid == 10) return hascells[t];
        if (tid == 11) return kstart[t];
        return 0;
    };
    auto put_meta = [&](int m, int reg) {
        if (tid < 8) S.nb[m][tid] = reg;
        else if (tid < 12) S.meta[m][tid - 8] = reg;  // cs, n (real cells), has, kstart
    };
    auto issue_role = [&](int b, int m, int has, int role) {
        if (role < 0) return;
        const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1, h = role >> 11;
        const int tt = S.nb[m][dp];
        if ((has || owned) && tt >= 0) {
            const int64_t n = (int64_t)tt * 64 + loc;
#pragma unroll
            for (int q = 0; q < (int)(sizeof(vec4<T>) / 16); q++)
                cp_async16(reinterpret_cast<char *>(&S.uh[b][h]) + 16 * q, reinterpret_cast<const char *>(u + n) + 16 * q);
            if (owned) cp_async_real<T>(&S.mh[b][loc], nmass + n);
        } else {
            S.uh[b][h] = mk4<T>(0, 0, 0, 0);
            if (owned) S.mh[b][loc] = T(0);
        }
    };
    T k[45];
    // tile t's tangent -> registers, its halo -> shared slot b (all threads, after its metadata is visible)
    auto issue = [&](int t, int b, int m) {
        if (t < T_) {
            const int cs = S.meta[m][0], ncp = S.meta[m][1], has = S.meta[m][2];
            const int cj = hvp_cell(tid), ks = hvp_slot(tid, ncp);
            if (has && cj < ncp) {
                const T *base = K + S.meta[m][3];
#pragma unroll
                for (int c = 0; c < NCH; c++) ldg_vec<T>(base + ((int64_t)c * ncp + ks) * VEC, k + c * VEC);
                k[44] = __ldg(base + (int64_t)NCH * VEC * ncp + ks);
            }
            if (has && tid * 4 < ncp) cp_async4(&S.cl[b][tid * 4], clocal + cs + tid * 4);
            issue_role(b, m, has, role0);
            issue_role(b, m, has, role1);
        }
        cp_async_commit();
    };
    put_meta(0, load_meta(t0));
    put_meta(1, load_meta(t0 + G));
    __syncthreads();
    issue(t0, 0, 0);
    int reg = load_meta(t0 + 2 * G);
    double acc = 0.0;
    int it = 0;
    for (int t = t0; t < T_; t += G, it++) {
        const int b = it & 1, m = it % 3;
        cp_async_wait<0>();
        __syncthreads();  // (B) halo slot b complete; metadata slot (it+1)%3 visible
        const int ncp = S.meta[m][1], has = S.meta[m][2];  // ncp: real cells of the tile
        const vec4<T> *uh = S.uh[b];
        const int cj = hvp_cell(tid);
        const int l = (has && cj < ncp) ? (int)S.cl[b][cj] : 0xFF;
        T P[9];
        int hb = 0;
        if (l != 0xFF) {
            const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
            hb = (lx * 5 + ly) * 5 + lz;
            T dG[9];
#pragma unroll
            for (int a = 0; a < 9; a++) dG[a] = T(0);
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                vec4<T> w = uh[hb + ox * 25 + oy * 5 + oz];
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
        // k is free: start the next tile's loads now; they overlap the scatter and node phase
        issue(t + G, b ^ 1, (it + 1) % 3);
        if (l != 0xFF) {
            T *Fw = S.F[tid >> 5][0];
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                const int h = hb + ox * 25 + oy * 5 + oz;
                Fw[h] += P[0] * s0 + P[1] * s1 + P[2] * s2;
                Fw[128 + h] += P[3] * s0 + P[4] * s1 + P[5] * s2;
                Fw[256 + h] += P[6] * s0 + P[7] * s1 + P[8] * s2;
                __syncwarp(__activemask());
            }
        }
        int64_t nidx[2];
        T fm[2][3];
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            nidx[r] = -1;
            fm[r][0] = fm[r][1] = fm[r][2] = T(0);
            if (role < 0) continue;
            const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1, h = role >> 11;
            if (!has && !owned) continue;
            const int tt = dp ? S.nb[m][dp] : t;
            if (tt < 0) continue;
            nidx[r] = (int64_t)tt * 64 + loc;
            if (owned) {
                const T mm = S.mh[b][loc];
                if (mm > T(0)) {
                    const vec4<T> w = uh[h];
                    fm[r][0] = mm * w.x; fm[r][1] = mm * w.y; fm[r][2] = mm * w.z;
                    acc += (double)(mm * (w.x * w.x + w.y * w.y + w.z * w.z));
                }
            }
        }
        __syncthreads();  // (C) F complete
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            if (role < 0) continue;
            const int h = role >> 11, interior = (role >> 10) & 1;
            const T f0 = S.F[0][0][h] + S.F[1][0][h] + fm[r][0], f1 = S.F[0][1][h] + S.F[1][1][h] + fm[r][1],
                    f2 = S.F[0][2][h] + S.F[1][2][h] + fm[r][2];
            S.F[0][0][h] = S.F[0][1][h] = S.F[0][2][h] = S.F[1][0][h] = S.F[1][1][h] = S.F[1][2][h] = T(0);
            if (nidx[r] < 0) continue;
            if (interior) Hu[nidx[r]] = mk4<T>(f0, f1, f2, T(0));
            else if (f0 != T(0) || f1 != T(0) || f2 != T(0)) atomic_add3<T>(Hu + nidx[r], f0, f1, f2);
        }
        put_meta((it + 2) % 3, reg);  // metadata of tile t + 2G (slot last read by tile t - G)
        reg = load_meta(t + 3 * G);
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

// ---------------------------------------------------------------------------------------------
// v5 (MPL_HVP_KERNEL=rq, default): rp with an instruction diet.  ncu of rp at cfg4: 72 M warp
// instructions (IPC 1.9), 42 % of them integer / control flow (divergence around inactive lanes and
// the masked scatter), shared-memory pipe 51 % busy with 2-way bank conflicts on a third of its
// wavefronts.  Changes:
//   * every lane has a distinct cell position: perm[t][j] lists the tile's cells, then its empty
//     positions, so lanes without a cell run the same code with dG = 0 (no divergence, full-warp
//     __syncwarp between scatter passes);
//   * dG and the 8 corner forces by tensor-product sums/differences (17 + 10 adds per component
//     instead of 24 + 24);
//   * shared layouts chosen (exhaustive search) so a full tile's 32 cells per warp hit distinct banks
//     in every pass: u halo at 5hx + 25hy + 2hz (16-byte slots, 129), forces at 8hx + 25hy + 10hz (173).
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr int rq_u(int hx, int hy, int hz) { return 5 * hx + 25 * hy + 2 * hz; }
__host__ __device__ constexpr int rq_f(int hx, int hy, int hz) { return 8 * hx + 25 * hy + 10 * hz; }
constexpr int RQ_U = 132, RQ_F = 176;

template <class T> struct RqSmem {
    alignas(16) vec4<T> uh[2][RQ_U];
    alignas(16) T mh[2][64];
    alignas(16) uint8_t pm[2][64];  // lane permutation of the tile (cp.async'ed with the halo)
    T F[2][3][RQ_F];
    int nb[3][8];
    int meta[3][4];  // cs, n (real cells), has, kstart
    double red[2];
};

// role: bits 0-5 local node id, 6-8 neighbour slot, 9 owned, 10 interior, 11-18 u slot, 19-26 F slot
__device__ __forceinline__ int rq_role(int h) {
    if (h >= 125) return -1;
    const int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
    const int dp = ((hx >> 2) << 2) | ((hy >> 2) << 1) | (hz >> 2);
    const int loc = local_id(hx & 3, hy & 3, hz & 3);
    const int interior = (hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3);
    return loc | (dp << 6) | ((dp == 0) << 9) | (interior << 10) | (rq_u(hx, hy, hz) << 11) | (rq_f(hx, hy, hz) << 19);
}

template <class T, int MINB>
__global__ void __launch_bounds__(64, MINB) k_hvp_rq(int T_, const int *__restrict__ nplus, const uint8_t *__restrict__ perm,
                                               const int *__restrict__ hascells, const T *__restrict__ K,
                                               const int *__restrict__ kstart, const int *__restrict__ ncell,
                                               const T *__restrict__ nmass, const vec4<T> *__restrict__ u,
                                               vec4<T> *__restrict__ Hu, double *__restrict__ uHu,
                                               const CGSlot *__restrict__ cgs, int cgj, double cgthr,
                                               const DevScalars *__restrict__ sc) {
    __shared__ RqSmem<T> S;
    const int tid = threadIdx.x;
    if (cgs != nullptr) {
        double rr = stripe_sum_bcast(cgs[cgj].rr);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    constexpr int VEC = KL<T>::VEC, NCH = KL<T>::NCH;
    const int role0 = rq_role(tid), role1 = rq_role(tid + 64);
    for (int i = tid; i < 2 * 3 * RQ_F; i += 64) (&S.F[0][0][0])[i] = T(0);
    const int G = gridDim.x, t0 = blockIdx.x;
    const int j = hvp_cell(tid);  // this lane's cell rank in every tile
    auto load_meta = [&](int t) -> int {
        if (t >= T_) return 0;
        if (tid < 8) return tid ? nplus[8 * t + tid] : t;
        if (tid == 9) return ncell[t];
        if (tid == 10) return hascells[t];
        if (tid == 11) return kstart[t];
        return 0;
    };
    auto put_meta = [&](int m, int reg) {
        if (tid < 8) S.nb[m][tid] = reg;
        else if (tid < 12) S.meta[m][tid - 8] = reg;
    };
    auto issue_role = [&](int b, int m, int has, int role) {
        if (role < 0) return;
        const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1, uo = (role >> 11) & 255;
        const int tt = S.nb[m][dp];
        if ((has || owned) && tt >= 0) {
            const int64_t n = (int64_t)tt * 64 + loc;
#pragma unroll
            for (int q = 0; q < (int)(sizeof(vec4<T>) / 16); q++)
                cp_async16(reinterpret_cast<char *>(&S.uh[b][uo]) + 16 * q, reinterpret_cast<const char *>(u + n) + 16 * q);
            if (owned) cp_async_real<T>(&S.mh[b][loc], nmass + n);
        } else {
            S.uh[b][uo] = mk4<T>(0, 0, 0, 0);
            if (owned) S.mh[b][loc] = T(0);
        }
    };
    T k[45];
#pragma unroll
    for (int i = 0; i < 45; i++) k[i] = T(0);
    int anext = 0;
    // tile t: tangent -> registers, lane permutation + halo -> shared slot b
    auto issue = [&](int t, int b, int m) {
        if (t < T_) {
            const int ncp = S.meta[m][1], has = S.meta[m][2];
            anext = has && j < ncp;
            if (tid < 4) {
                if (has) cp_async16(&S.pm[b][16 * tid], perm + (int64_t)t * 64 + 16 * tid);
                else
                    for (int q = 0; q < 16; q++) S.pm[b][16 * tid + q] = (uint8_t)(16 * tid + q);
            }
            if (anext) {
                // 32-bit element offsets from the tile's block (a block is < 64 x 45 reals)
                const T *blk = K + S.meta[m][3];
                const int sl = hvp_slot(tid, ncp);
                int off = sl * VEC;
#pragma unroll
                for (int c = 0; c < NCH; c++, off += ncp * VEC) ldg_vec<T>(blk + off, k + c * VEC);
                k[44] = __ldg(blk + NCH * VEC * ncp + sl);
            }
            issue_role(b, m, has, role0);
            issue_role(b, m, has, role1);
        }
        cp_async_commit();
    };
    put_meta(0, load_meta(t0));
    put_meta(1, load_meta(t0 + G));
    __syncthreads();
    issue(t0, 0, 0);
    int reg = load_meta(t0 + 2 * G);
    double acc = 0.0;
    int b = 0, m = 0;
    for (int t = t0; t < T_; t += G) {
        cp_async_wait<0>();
        __syncthreads();  // (B) halo slot b complete; metadata slot m+1 visible
        const int has = S.meta[m][2];
        const int l = S.pm[b][j];
        const T am = anext ? T(1) : T(0);
        const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
        const vec4<T> *uh = S.uh[b] + rq_u(lx, ly, lz);
        T dG[9];
        {
            vec4<T> w[8];
#pragma unroll
            for (int o = 0; o < 8; o++) w[o] = uh[rq_u((o >> 2) & 1, (o >> 1) & 1, o & 1)];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                T c[8];
#pragma unroll
                for (int o = 0; o < 8; o++) c[o] = a == 0 ? w[o].x : (a == 1 ? w[o].y : w[o].z);
                // o = 4 ox + 2 oy + oz
                const T p00 = c[1] + c[0], m00 = c[1] - c[0], p01 = c[3] + c[2], m01 = c[3] - c[2];
                const T p10 = c[5] + c[4], m10 = c[5] - c[4], p11 = c[7] + c[6], m11 = c[7] - c[6];
                const T pp0 = p01 + p00, pm0 = p01 - p00, mp0 = m01 + m00;
                const T pp1 = p11 + p10, pm1 = p11 - p10, mp1 = m11 + m10;
                dG[3 * a + 0] = (pp1 - pp0) * am;
                dG[3 * a + 1] = (pm1 + pm0) * am;
                dG[3 * a + 2] = (mp1 + mp0) * am;
            }
        }
        T P[9];
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
        // k is free: the next tile's loads overlap the scatter and the node phase
        const int bn = b ^ 1, mn = m == 2 ? 0 : m + 1;
        issue(t + G, bn, mn);
        {
            T *Fw = S.F[tid >> 5][0] + rq_f(lx, ly, lz);
            T ypp[3], ypm[3];
#pragma unroll
            for (int a = 0; a < 3; a++) { ypp[a] = P[3 * a + 1] + P[3 * a + 2]; ypm[a] = P[3 * a + 1] - P[3 * a + 2]; }
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                const int fo = rq_f(ox, oy, oz);
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const T yz = oy ? (oz ? ypp[a] : ypm[a]) : (oz ? -ypm[a] : -ypp[a]);
                    Fw[a * RQ_F + fo] += (ox ? P[3 * a] : -P[3 * a]) + yz;
                }
                __syncwarp();
            }
        }
        int64_t nidx[2];
        T fm[2][3];
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            nidx[r] = -1;
            fm[r][0] = fm[r][1] = fm[r][2] = T(0);
            if (role < 0) continue;
            const int loc = role & 63, dp = (role >> 6) & 7, owned = (role >> 9) & 1;
            if (!has && !owned) continue;
            const int tt = dp ? S.nb[m][dp] : t;
            if (tt < 0) continue;
            nidx[r] = (int64_t)tt * 64 + loc;
            if (owned) {
                const T mm = S.mh[b][loc];
                const vec4<T> w = S.uh[b][(role >> 11) & 255];
                fm[r][0] = mm * w.x; fm[r][1] = mm * w.y; fm[r][2] = mm * w.z;
                acc += (double)(mm * (w.x * w.x + w.y * w.y + w.z * w.z));
            }
        }
        __syncthreads();  // (C) F complete
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int role = r ? role1 : role0;
            if (role < 0) continue;
            const int fo = (role >> 19) & 255, interior = (role >> 10) & 1;
            T f[3];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                f[a] = S.F[0][a][fo] + S.F[1][a][fo] + fm[r][a];
                S.F[0][a][fo] = T(0);
                S.F[1][a][fo] = T(0);
            }
            if (nidx[r] < 0) continue;
            if (interior) Hu[nidx[r]] = mk4<T>(f[0], f[1], f[2], T(0));
            else if (f[0] != T(0) || f[1] != T(0) || f[2] != T(0)) atomic_add3<T>(Hu + nidx[r], f[0], f[1], f[2]);
        }
        const int m2 = mn == 2 ? 0 : mn + 1;
        put_meta(m2, reg);  // metadata of tile t + 2G (slot last read by tile t - G)
        reg = load_meta(t + 3 * G);
        b = bn;
        m = mn;
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

int g_num_sms = 0;

template <class T, int MINB>
mpl_status launch_rq(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                     double cgthr) {
    static int per_sm[2] = {0, 0};
    const int pi = sizeof(T) == 8;
    if (per_sm[pi] == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_rq<T, MINB>, 64, 0));
        per_sm[pi] = occ > 0 ? occ : 1;
    }
    int grid = g_num_sms * per_sm[pi];
    if (grid > ctx->T) grid = ctx->T;
    k_hvp_rq<T, MINB><<<grid, 64, 0, ctx->stream>>>(
        ctx->T, (const int *)ctx->t_nplus.p, (const uint8_t *)ctx->t_perm.p, (const int *)ctx->t_hascells.p,
        (const T *)ctx->K.p, (const int *)ctx->t_kstart.p, (const int *)ctx->t_ncell.p, (const T *)owned_mass(ctx),
        (const vec4<T> *)u_tile, (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
    ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

template <class T, int MINB>
mpl_status launch_rp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                     double cgthr) {
    static int per_sm[2] = {0, 0};
    const int pi = sizeof(T) == 8;
    if (per_sm[pi] == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_rp<T, MINB>, 64, 0));
        per_sm[pi] = occ > 0 ? occ : 1;
    }
    int grid = g_num_sms * per_sm[pi];
    if (grid > ctx->T) grid = ctx->T;
    k_hvp_rp<T, MINB><<<grid, 64, 0, ctx->stream>>>(
        ctx->T, (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
        (const int *)ctx->t_hascells.p, (const T *)ctx->K.p, (const int *)ctx->t_kstart.p,
        (const int *)ctx->t_ncell.p, (const T *)owned_mass(ctx), (const vec4<T> *)u_tile,
        (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
    ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

template <class T, int NS>
mpl_status launch_pipe(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                       double cgthr) {
    static int per_sm[2] = {0, 0};
    const int pi = sizeof(T) == 8;
    const size_t smem = sizeof(PipeSmem<T, NS>);
    if (per_sm[pi] == 0) {
        MPL_CUDA(cudaFuncSetAttribute(k_hvp_pipe<T, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_pipe<T, NS>, 64, smem));
        per_sm[pi] = occ > 0 ? occ : 1;
    }
    int grid = g_num_sms * per_sm[pi];
    if (grid > ctx->T) grid = ctx->T;
    k_hvp_pipe<T, NS><<<grid, 64, smem, ctx->stream>>>(
        ctx->T, (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
        (const int *)ctx->t_hascells.p, (const T *)ctx->K.p, (const int *)ctx->t_kstart.p,
        (const int *)ctx->t_ncell.p, (const T *)owned_mass(ctx), (const vec4<T> *)u_tile,
        (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
    ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

}  // namespace

// Hu (tile-dense) must be zero on every node that receives atomics (all non-interior nodes).
template <class T>
mpl_status launch_hvp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                      double cgthr) {
    if (ctx->T == 0) return MPL_OK;
    static int variant = -1;
    if (variant < 0) {
        // "rp10" (default) / "rp" / "rp12": persistent, tangent register-pipelined (v4) with >= 10 / 1 /
        // 12 CTAs per SM requested from ptxas; "pipe2" / "pipe3": persistent TMA-ring v3 with 2 / 3
        // stages; "reg": one tile per CTA (v2)
        const char *e = getenv("MPL_HVP_KERNEL");
        variant = 5;
        if (e && e[0] == 'r' && e[1] == 'q') variant = e[2] == '8' ? 8 : 7;
        else if (e && e[0] == 'r' && e[1] == 'p') variant = e[2] == '1' ? (e[3] == '2' ? 6 : 5) : 4;
        else if (e && e[0] == 'r') variant = 0;
        else if (e && e[0] == 'p' && e[4] == '3') variant = 3;
    }
    if (variant == 7) return launch_rq<T, 10>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 8) return launch_rq<T, 8>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 2) return launch_pipe<T, 2>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 4) return launch_rp<T, 1>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 5) return launch_rp<T, 10>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 6) return launch_rp<T, 12>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 3) return launch_pipe<T, 3>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
    if (variant == 0) {
        k_hvp_reg<T><<<ctx->T, 64, 0, ctx->stream>>>(
            (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
            (const int *)ctx->t_hascells.p, (const T *)ctx->K.p, (const int *)ctx->t_kstart.p,
        (const int *)ctx->t_ncell.p, (const T *)owned_mass(ctx), (const vec4<T> *)u_tile,
            (vec4<T> *)Hu_tile, uHu, cgs, cgj, cgthr, (const DevScalars *)ctx->scalars.p);
        ctx->launches++;
        MPL_CUDA(cudaGetLastError());
    }
    return MPL_OK;
}

template mpl_status launch_hvp<float>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double);
template mpl_status launch_hvp<double>(mpl_ctx, const void *, void *, double *, const CGSlot *, int, double);
