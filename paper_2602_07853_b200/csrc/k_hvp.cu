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

// ---------------------------------------------------------------------------------------------
// v6 (MPL_HVP_KERNEL=wz, fp32 default): one warp per tile, two z-adjacent cells per lane, no block
// barriers.  ncu of rp10 at cfg4: 72 M warp instructions at IPC 1.9 — about 650 per warp per tile,
// three times the arithmetic — so the kernel was issue bound, not HBM bound.  Here:
//   * lane = 16 zp + 4 lx + ly owns cells A = (lx, ly, 2zp) and B = (lx, ly, 2zp + 1); they share the
//     4 nodes of the plane z = 2zp + 1, so the lane reads 12 node vectors instead of 16 and scatters
//     into 12 nodes instead of 16;
//   * dG of both cells by tensor-product sums per node plane (7 adds per plane and component);
//   * corner forces from 4 distinct sums per component and cell, signs folded into the adds;
//   * the tangent uses the "kz" slot order (kz_key): the A cells of a tile first, then the B cells,
//     each in lane order, so a warp's 16-byte loads of one chunk are contiguous; the 90 tangent
//     numbers of the next tile are loaded (L2 evict-first) as soon as the current tile's K dG is done;
//   * the u halo (shared slot 5x + 26y + z: conflict-free 16-byte accesses for every quarter-warp)
//     and the owned masses are cp.async double-buffered per warp; the 12 scatter passes are
//     read-modify-writes of a per-warp force buffer in the same slot map, separated by __syncwarp
//     only (each pass is injective over the lanes).
// ---------------------------------------------------------------------------------------------
constexpr int WZ_W = 4;  // independent warps per CTA
// per-warp shared state; PLANE: the 12 scatter passes write non-aliasing planes pl[pass][lane] (no
// read-modify-write chain), the node phase sums a node's <= 8 plane entries
template <bool PLANE> struct WzWarp {
    alignas(16) f4 uh[2][132];
    alignas(16) f4 F[PLANE ? 12 * 32 : 132];
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
// PLANE gather of node (X, Y, Z): pass (ox, oy, q) of lane (X - ox, Y - oy, zp) with 2 zp + q = Z lands
// at pl index ((2 ox + oy) 3 + q) 32 + 16 zp + 4 (X - ox) + (Y - oy) = base + zoff + 188 ox + 95 oy,
// base = 4X + Y.  Encoded: base | zoff1 << 5 | (Z == 2: second entry zoff 16) << 12 | valid (ox, oy)
// mask << 13 (bit 2 ox + oy)
__device__ __forceinline__ int wz_gather(int n) {
    if (n >= 125) return 0;
    int X, Y, Z;
    wz_node(n, X, Y, Z);
    const int zoff1 = Z == 0 ? 0 : Z == 1 ? 32 : Z == 2 ? 64 : Z == 3 ? 48 : 80;
    int mask = 0;
    for (int ox = 0; ox < 2; ox++)
        for (int oy = 0; oy < 2; oy++)
            if (X - ox >= 0 && X - ox <= 3 && Y - oy >= 0 && Y - oy <= 3) mask |= 1 << (2 * ox + oy);
    return (4 * X + Y) | (zoff1 << 5) | ((Z == 2) << 12) | (mask << 13);
}

// packed upper-triangle element e -> row r (kofs(r) <= e < kofs(r + 1)) and column
__host__ __device__ constexpr int krow(int e) {
    int r = 0;
    while (r < 8 && kofs(r + 1) <= e) r++;
    return r;
}
__host__ __device__ constexpr int kcol(int e) { return krow(e) + (e - kofs(krow(e))); }

// ROLL: each 16-byte chunk of the next tile's tangent is requested as soon as the current tile's K dG
// has consumed its registers (a whole tile period to arrive) instead of after the whole K dG.
// SCAT: how the 12 node contributions of a lane reach the nodes —
//   WZ_RMW   read-modify-write passes into a per-warp force buffer, then a node phase (4 nodes / lane);
//   WZ_PLANE non-aliasing plane stores, node phase sums <= 8 plane entries per node;
//   WZ_SHFL  register reduction with shuffles along y (1 lane), x (4 lanes), z (16 lanes), after which
//            every node value sits in exactly one (lane, slot) and goes straight to global memory; no
//            force buffer and no node phase;
//   WZ_RMW3  WZ_RMW with the z = 2 plane merged by a shuffle first, so the passes form 4 groups of 3
//            non-aliasing read-modify-writes.
enum { WZ_RMW = 0, WZ_PLANE = 1, WZ_SHFL = 2, WZ_RMW3 = 3 };
template <int MINB, bool ROLL, int SCAT, bool PAD>
__global__ void __launch_bounds__(32 * WZ_W, MINB)
    k_hvp_wz(int T_, const int *__restrict__ nplus, const unsigned long long *__restrict__ cmask,
             const int *__restrict__ hascells, const float *__restrict__ K, const int *__restrict__ kstart,
             const float *__restrict__ nmass, const f4 *__restrict__ u, f4 *__restrict__ Hu, double *__restrict__ uHu,
             const CGSlot *__restrict__ cgs, int cgj, double cgthr, const DevScalars *__restrict__ sc) {
    constexpr bool PLANE = SCAT == WZ_PLANE, SHFL = SCAT == WZ_SHFL;
    __shared__ WzWarp<PLANE> SW[WZ_W];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WzWarp<PLANE> &S = SW[wid];
    pdl_trigger();
    pdl_wait();
    if (cgs != nullptr) {
        const double rr = warp_sum(cgs[cgj].rr[lane]);
        if (sc->neg_curv || (cgj > 0 && rr <= cgthr)) return;
    }
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    const int zp = lane >> 4, lx = (lane >> 2) & 3, ly = lane & 3;
    const int lA = lx * 16 + ly * 4 + 2 * zp;  // cell A's local position (B = lA + 1)
    const int hb = 5 * lx + 26 * ly + 2 * zp;  // u-halo slot of cell A's (0,0,0) corner
    int role[4], gat[4];
#pragma unroll
    for (int r = 0; r < 4; r++) { role[r] = wz_role(lane + 32 * r); gat[r] = PLANE ? wz_gather(lane + 32 * r) : 0; }
    if (SCAT == WZ_RMW)
        for (int i = lane; i < 132; i += 32) S.F[i] = mk4<float>(0.f, 0.f, 0.f, 0.f);
    const uint64_t pol = l2_evict_first_policy();
    const int G = gridDim.x * WZ_W, t0 = blockIdx.x * WZ_W + wid;
    // tile metadata, spread over lanes 0-11: neighbours (lane 0 = the tile itself), kstart, has, cmask
    // halves; one 32-bit load per lane at a per-lane base + stride t, no use until the next iteration
    const int *mbase = lane < 8 ? nplus + lane : lane == 8 ? kstart : lane == 9 ? hascells
                                                                      : reinterpret_cast<const int *>(cmask) + (lane - 10);
    const int mstride = lane < 8 ? 8 : lane < 10 ? 1 : 2;
    auto load_meta = [&](int t) -> int {
        if (t >= T_ || lane >= 12) return 0;
        return lane == 0 ? t : __ldg(mbase + (int64_t)mstride * t);
    };
    struct TileK {
        int has, pA, pB;         // the tile has cells; this lane's cells A / B are present
        unsigned sb;             // compact: chunk stride in bytes (16 n)
        int e44, d44;            // compact: element 44 of cell A at ka + e44, of cell B at kbp + e44 - 3 d44
        const float *ka, *kbp;   // this lane's first chunk of cell A / B (PAD: cell A; B at + 128)
    };
    auto tile_k = [&](int t, int meta) -> TileK {
        TileK q;
        q.has = __shfl_sync(FULL, meta, 9);
        const int ks = __shfl_sync(FULL, meta, 8);
        const unsigned clo = (unsigned)__shfl_sync(FULL, meta, 10), chi = (unsigned)__shfl_sync(FULL, meta, 11);
        if (t >= T_) q.has = 0;
        const unsigned word = lA < 32 ? clo : chi;
        q.pA = q.has ? (int)((word >> (lA & 31)) & 1u) : 0;
        q.pB = q.has ? (int)((word >> ((lA + 1) & 31)) & 1u) : 0;
        if (PAD) {
            q.ka = K + ks + 4 * lane;
        } else {
            const unsigned pmA = __ballot_sync(FULL, q.pA), pmB = __ballot_sync(FULL, q.pB);
            const int nA = __popc(pmA), n = nA + __popc(pmB);
            const int sA = __popc(pmA & lt), sB = nA + __popc(pmB & lt);
            q.sb = 16u * (unsigned)n;
            q.ka = K + ks + 4 * sA;
            q.kbp = K + ks + 4 * sB;
            q.e44 = 44 * n + sA - 4 * sA;  // element 44 of slot s at 44 n + s, relative to ka / kbp
            q.d44 = sB - sA;
        }
        return q;
    };
    float k[90];
    // chunk c < 11 of slot s at 4 (c n + s), element 44 at 44 n + s (k_off); PAD: n = 64, cell A in slot
    // lane, cell B in slot 32 + lane, so every load is an immediate offset from q.ka; compact: chunk c at
    // (byte) ka + c * 16 n, one IMAD.WIDE per load.  Chunk c of cell X (off 0 = A, 45 = B) -> k
    auto kload = [&](const TileK &q, int off, int c) {
        if (!(off ? q.pB : q.pA)) return;
        if (PAD) {
            const float *p = q.ka + (off ? 128 : 0);
            if (c < 11) {
                const float4 v = ldg_stream(p + 256 * c, pol);
                k[off + 4 * c] = v.x; k[off + 4 * c + 1] = v.y; k[off + 4 * c + 2] = v.z; k[off + 4 * c + 3] = v.w;
            } else {
                k[off + 44] = ldg_stream1(p - 3 * lane - (off ? 96 : 0) + 2816, pol);
            }
        } else {
            const float *p = off ? q.kbp : q.ka;
            if (c < 11) {
                const float4 v = ldg_stream(reinterpret_cast<const float *>(reinterpret_cast<const char *>(p) +
                                                                            (uint64_t)q.sb * (uint64_t)c), pol);
                k[off + 4 * c] = v.x; k[off + 4 * c + 1] = v.y; k[off + 4 * c + 2] = v.z; k[off + 4 * c + 3] = v.w;
            } else {
                k[off + 44] = ldg_stream1(p + q.e44 - (off ? 3 * q.d44 : 0), pol);
            }
        }
    };
    // tile t: u halo + owned masses -> shared buffer b (cp.async, one group)
    auto halo = [&](int t, int b, int meta) {
        const int has = __shfl_sync(FULL, meta, 9);
        int tt[4];
#pragma unroll
        for (int r = 0; r < 4; r++) tt[r] = __shfl_sync(FULL, meta, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
        if (t < T_) {
#pragma unroll
            for (int r = 0; r < 4; r++) {
                if (role[r] < 0) continue;
                const int loc = role[r] & 63, owned = (role[r] >> 9) & 1, h = role[r] >> 11;
                if ((has || owned) && tt[r] >= 0) {
                    const int64_t nd = (int64_t)tt[r] * 64 + loc;
                    cp_async16(&S.uh[b][h], u + nd);
                    if (owned) cp_async4(&S.mh[b][loc], nmass + nd);
                } else {
                    S.uh[b][h] = mk4<float>(0.f, 0.f, 0.f, 0.f);
                    if (owned) S.mh[b][loc] = 0.f;
                }
            }
        }
        cp_async_commit();
    };
    int mcur = load_meta(t0);
    int mnext = load_meta(t0 + G);
    TileK cur = tile_k(t0, mcur);
#pragma unroll
    for (int c = 0; c < 12; c++) { kload(cur, 0, c); kload(cur, 45, c); }
    halo(t0, 0, mcur);
    double acc = 0.0;
    int it = 0;
    for (int t = t0; t < T_; t += G, it++) {
        const int b = it & 1;
        const int mnn = load_meta(t + 2 * G);
        const TileK nxt = tile_k(t + G, mnext);
        cp_async_wait<0>();
        __syncwarp();
        const f4 *uh = S.uh[b];
        float PA[9], PB[9];
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
            // ---- P = K dG (symmetric, packed upper triangle), element by element
#pragma unroll
            for (int r = 0; r < 9; r++) { PA[r] = 0.f; PB[r] = 0.f; }
#pragma unroll
            for (int e = 0; e < 45; e++) {
                const int r = krow(e), c = kcol(e);
                PA[r] += k[e] * dA[c];
                if (c != r) PA[c] += k[e] * dA[r];
                if (ROLL && ((e & 3) == 3 || e == 44)) kload(nxt, 0, e >> 2);
            }
#pragma unroll
            for (int e = 0; e < 45; e++) {
                const int r = krow(e), c = kcol(e);
                PB[r] += k[45 + e] * dB[c];
                if (c != r) PB[c] += k[45 + e] * dB[r];
                if (ROLL && ((e & 3) == 3 || e == 44)) kload(nxt, 45, e >> 2);
            }
            float qf = 0.f;
#pragma unroll
            for (int r = 0; r < 9; r++) {
                PA[r] = cur.pA ? PA[r] : 0.f;  // absent cells: k holds stale numbers
                PB[r] = cur.pB ? PB[r] : 0.f;
                qf += PA[r] * dA[r] + PB[r] * dB[r];
            }
            acc += (double)qf;
        }
        // SHFL without ROLL: the next tile's tangent is requested after the register reduction, so k's
        // registers can hold the 36 node contributions meanwhile
        constexpr bool LATE = SHFL && !ROLL;
        if (!LATE && (!ROLL || !cur.has)) {
            // k is free: start the next tile's loads; they overlap the scatter and the node phase
#pragma unroll
            for (int c = 0; c < 12; c++) { kload(nxt, 0, c); kload(nxt, 45, c); }
        }
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
        if (SHFL) {
            // ---- contributions c[ox][oy][q] of node (lx + ox, ly + oy, 2 zp + q), reduced in registers
            float c[2][2][3][3];
            if (cur.has) {
                float gA[3][4], gB[3][4];
#pragma unroll
                for (int a = 0; a < 3; a++) {
                    const float e1 = PA[3 * a] + PA[3 * a + 1], e2 = PA[3 * a] - PA[3 * a + 1], z = PA[3 * a + 2];
                    gA[a][0] = e1 + z; gA[a][1] = e1 - z; gA[a][2] = e2 + z; gA[a][3] = e2 - z;
                    const float f1 = PB[3 * a] + PB[3 * a + 1], f2 = PB[3 * a] - PB[3 * a + 1], y = PB[3 * a + 2];
                    gB[a][0] = f1 + y; gB[a][1] = f1 - y; gB[a][2] = f2 + y; gB[a][3] = f2 - y;
                }
#pragma unroll
                for (int ox = 0; ox < 2; ox++)
#pragma unroll
                    for (int oy = 0; oy < 2; oy++)
#pragma unroll
                        for (int q = 0; q < 3; q++)
#pragma unroll
                            for (int a = 0; a < 3; a++) {
                                float v = 0.f;
                                if (q < 2) v = corner(gA[a], ox, oy, q);
                                if (q > 0) v += corner(gB[a], ox, oy, q - 1);
                                c[ox][oy][q][a] = v;
                            }
                // y: node (., ly + 1, .) of lane ly == node (., ly, .) of lane ly + 1
#pragma unroll
                for (int ox = 0; ox < 2; ox++)
#pragma unroll
                    for (int q = 0; q < 3; q++)
#pragma unroll
                        for (int a = 0; a < 3; a++) {
                            const float r = __shfl_up_sync(FULL, c[ox][1][q][a], 1);
                            if (ly > 0) c[ox][0][q][a] += r;
                        }
                // x: 4 lanes
#pragma unroll
                for (int oy = 0; oy < 2; oy++)
#pragma unroll
                    for (int q = 0; q < 3; q++)
#pragma unroll
                        for (int a = 0; a < 3; a++) {
                            const float r = __shfl_up_sync(FULL, c[1][oy][q][a], 4);
                            if (lx > 0) c[0][oy][q][a] += r;
                        }
                // z: plane q = 2 of zp = 0 is plane q = 0 of zp = 1
#pragma unroll
                for (int ox = 0; ox < 2; ox++)
#pragma unroll
                    for (int oy = 0; oy < 2; oy++)
#pragma unroll
                        for (int a = 0; a < 3; a++) {
                            const float r = __shfl_up_sync(FULL, c[ox][oy][2][a], 16);
                            if (zp > 0) c[ox][oy][0][a] += r;
                        }
            } else {
#pragma unroll
                for (int i = 0; i < 36; i++) (&c[0][0][0][0])[i] = 0.f;
            }
            if (LATE) {
#pragma unroll
                for (int cc = 0; cc < 12; cc++) { kload(nxt, 0, cc); kload(nxt, 45, cc); }
            }
            // ---- outputs: slot (ox, oy, q) holds a complete node iff (ox == 0 || lx == 3) && (oy == 0 ||
            // ly == 3) && (q < 2 || zp == 1); its tile is neighbour (ox, oy, q == 2) (warp-uniform)
#pragma unroll
            for (int ox = 0; ox < 2; ox++)
#pragma unroll
                for (int oy = 0; oy < 2; oy++)
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const int dp = (ox << 2) | (oy << 1) | (q == 2);
                        const int tt = __shfl_sync(FULL, mcur, dp);
                        const bool valid = (ox == 0 || lx == 3) && (oy == 0 || ly == 3) && (q < 2 || zp == 1);
                        if (!valid || tt < 0) continue;
                        const int X = lx + ox, Y = ly + oy, Z = 2 * zp + q;
                        const int loc = local_id(X & 3, Y & 3, Z & 3);
                        float fx = c[ox][oy][q][0], fy = c[ox][oy][q][1], fz = c[ox][oy][q][2];
                        bool interior = false;
                        if (dp == 0) {  // owned node: lumped mass term
                            const float mm = S.mh[b][loc];
                            if (mm > 0.f) {
                                const f4 w = uh[hb + q];
                                fx += mm * w.x; fy += mm * w.y; fz += mm * w.z;
                                acc += (double)(mm * (w.x * w.x + w.y * w.y + w.z * w.z));
                            }
                            interior = X >= 1 && Y >= 1 && Z >= 1 && Z <= 3;
                        } else if (!cur.has) {
                            continue;
                        }
                        const int64_t nd = (int64_t)tt * 64 + loc;
                        if (interior) Hu[nd] = mk4<float>(fx, fy, fz, 0.f);
                        else if (fx != 0.f || fy != 0.f || fz != 0.f) atomic_add3<float>(Hu + nd, fx, fy, fz);
                    }
            __syncwarp();  // uh[b] / mh[b] read before the next halo refills them
            mcur = mnext;
            mnext = mnn;
            cur = nxt;
            continue;
        }
        if (cur.has) {
            float gA[3][4], gB[3][4];
#pragma unroll
            for (int a = 0; a < 3; a++) {
                const float e1 = PA[3 * a] + PA[3 * a + 1], e2 = PA[3 * a] - PA[3 * a + 1], z = PA[3 * a + 2];
                gA[a][0] = e1 + z; gA[a][1] = e1 - z; gA[a][2] = e2 + z; gA[a][3] = e2 - z;
                const float f1 = PB[3 * a] + PB[3 * a + 1], f2 = PB[3 * a] - PB[3 * a + 1], y = PB[3 * a + 2];
                gB[a][0] = f1 + y; gB[a][1] = f1 - y; gB[a][2] = f2 + y; gB[a][3] = f2 - y;
            }
            if (SCAT == WZ_RMW3) {
                // plane z = 2 is q = 2 of the zp = 0 lanes and q = 0 of the zp = 1 lanes: merge it with a
                // shuffle, after which the q = 0 (z = 0, 2), q = 1 (z = 1, 3) and q = 2 (z = 4, zp = 1 only)
                // passes touch disjoint nodes; 4 groups of 3 independent read-modify-writes, one
                // __syncwarp per group instead of one per pass
                float zr[2][2][3];
#pragma unroll
                for (int ox = 0; ox < 2; ox++)
#pragma unroll
                    for (int oy = 0; oy < 2; oy++)
#pragma unroll
                        for (int a = 0; a < 3; a++) {
                            const float v = __shfl_up_sync(FULL, corner(gB[a], ox, oy, 1), 16);
                            zr[ox][oy][a] = zp ? v : 0.f;
                        }
#pragma unroll
                for (int ox = 0; ox < 2; ox++)
#pragma unroll
                    for (int oy = 0; oy < 2; oy++) {
                        f4 *f0 = &S.F[hb + 5 * ox + 26 * oy];
                        // the first group touching a node stores instead of adding (no zeroing pass)
                        const bool first = (ox == 0 || lx == 3) && (oy == 0 || ly == 3);
                        const f4 zero4 = mk4<float>(0.f, 0.f, 0.f, 0.f);
                        const f4 o0 = first ? zero4 : f0[0], o1 = first ? zero4 : f0[1];
                        f0[0] = mk4<float>(o0.x + corner(gA[0], ox, oy, 0) + zr[ox][oy][0],
                                           o0.y + corner(gA[1], ox, oy, 0) + zr[ox][oy][1],
                                           o0.z + corner(gA[2], ox, oy, 0) + zr[ox][oy][2], 0.f);
                        f0[1] = mk4<float>(o1.x + corner(gA[0], ox, oy, 1) + corner(gB[0], ox, oy, 0),
                                           o1.y + corner(gA[1], ox, oy, 1) + corner(gB[1], ox, oy, 0),
                                           o1.z + corner(gA[2], ox, oy, 1) + corner(gB[2], ox, oy, 0), 0.f);
                        if (zp) {
                            const f4 o2 = first ? zero4 : f0[2];
                            f0[2] = mk4<float>(o2.x + corner(gB[0], ox, oy, 1), o2.y + corner(gB[1], ox, oy, 1),
                                               o2.z + corner(gB[2], ox, oy, 1), 0.f);
                        }
                        __syncwarp();
                    }
            } else
#pragma unroll
            for (int ox = 0; ox < 2; ox++)
#pragma unroll
                for (int oy = 0; oy < 2; oy++)
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        f4 f = mk4<float>(0.f, 0.f, 0.f, 0.f);
                        if (q < 2) { f.x = corner(gA[0], ox, oy, q); f.y = corner(gA[1], ox, oy, q); f.z = corner(gA[2], ox, oy, q); }
                        if (q > 0) {
                            f.x += corner(gB[0], ox, oy, q - 1); f.y += corner(gB[1], ox, oy, q - 1);
                            f.z += corner(gB[2], ox, oy, q - 1);
                        }
                        if (PLANE) {
                            S.F[((2 * ox + oy) * 3 + q) * 32 + lane] = f;
                        } else {
                            f4 *fp = &S.F[hb + 5 * ox + 26 * oy + q];
                            const f4 o = *fp;
                            *fp = mk4<float>(o.x + f.x, o.y + f.y, o.z + f.z, 0.f);
                            __syncwarp();
                        }
                    }
            if (PLANE) __syncwarp();
        }
        // ---- node phase: forces + lumped mass term, stored (interior) or added atomically (faces)
        int tt[4];
#pragma unroll
        for (int r = 0; r < 4; r++) tt[r] = __shfl_sync(FULL, mcur, role[r] < 0 ? 0 : (role[r] >> 6) & 7);
#pragma unroll
        for (int r = 0; r < 4; r++) {
            if (role[r] < 0) continue;
            const int loc = role[r] & 63, owned = (role[r] >> 9) & 1, interior = (role[r] >> 10) & 1,
                      h = role[r] >> 11;
            f4 f = mk4<float>(0.f, 0.f, 0.f, 0.f);
            if (cur.has) {
                if (PLANE) {
                    const int g = gat[r], i1 = (g & 31) + ((g >> 5) & 127), two = (g >> 12) & 1, mk = g >> 13;
#pragma unroll
                    for (int o = 0; o < 4; o++) {
                        if (!((mk >> o) & 1)) continue;
                        const int i = i1 + (o >> 1) * 188 + (o & 1) * 95;
                        const f4 a = S.F[i];
                        f.x += a.x; f.y += a.y; f.z += a.z;
                        if (two) {
                            const f4 c2 = S.F[i - 48];  // zoff 64 -> 16
                            f.x += c2.x; f.y += c2.y; f.z += c2.z;
                        }
                    }
                } else {
                    f = S.F[h];
                    if (SCAT == WZ_RMW) S.F[h] = mk4<float>(0.f, 0.f, 0.f, 0.f);  // RMW3: first writers store
                }
            }
            if (!(cur.has || owned) || tt[r] < 0) continue;
            if (owned) {
                const float mm = S.mh[b][loc];
                if (mm > 0.f) {
                    const f4 w = uh[h];
                    f.x += mm * w.x; f.y += mm * w.y; f.z += mm * w.z;
                    acc += (double)(mm * (w.x * w.x + w.y * w.y + w.z * w.z));
                }
            }
            const int64_t nd = (int64_t)tt[r] * 64 + loc;
            if (interior) Hu[nd] = mk4<float>(f.x, f.y, f.z, 0.f);
            else if (f.x != 0.f || f.y != 0.f || f.z != 0.f) atomic_add3<float>(Hu + nd, f.x, f.y, f.z);
        }
        __syncwarp();  // node phase done reading uh[b] / mh[b] / planes before they are refilled
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

template <int MINB, bool ROLL, int SCAT, bool PAD>
mpl_status launch_wz(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                     double cgthr) {
    static int per_sm = 0;
    if (per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        MPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hvp_wz<MINB, ROLL, SCAT, PAD>, 32 * WZ_W, 0));
        per_sm = occ > 0 ? occ : 1;
    }
    int grid = g_num_sms * per_sm;
    const int need = (ctx->T + WZ_W - 1) / WZ_W;
    if (grid > need) grid = need;
    MPL_CUDA(launch_pdl(k_hvp_wz<MINB, ROLL, SCAT, PAD>, grid, 32 * WZ_W, 0, ctx->stream, ctx->T,
                        (const int *)ctx->t_nplus.p, (const unsigned long long *)ctx->t_cmask.p,
                        (const int *)ctx->t_hascells.p, (const float *)ctx->K.p, (const int *)ctx->t_kstart.p,
                        (const float *)owned_mass(ctx), (const f4 *)u_tile, (f4 *)Hu_tile, uHu, cgs, cgj, cgthr,
                        (const DevScalars *)ctx->scalars.p));
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

// HVP variant from MPL_HVP_KERNEL: "wh" / "wh4" (half-tile warps, v7), "wz" (default for fp32; fp64
// falls back to rp10; "wzp" with the
// plane scatter, "wzs" with the shuffle reduction, "wz2" / "wzp2" / "wzs2" with rolling tangent loads at
// 2 CTAs per SM), "rp10" (default
// for fp64), "rp" / "rp12": persistent, tangent register-pipelined (v4) with >= 10 / 1 / 12 CTAs per SM
// requested from ptxas; "rq" / "rq8" (v5); "pipe2" / "pipe3": persistent TMA-ring v3 with 2 / 3 stages;
// "reg": one tile per CTA (v2)
int hvp_variant() {
    static int variant = -1;
    if (variant < 0) {
        const char *e = getenv("MPL_HVP_KERNEL");
        variant = 11;
        if (e && e[0] == 'w' && e[1] == 'h') variant = e[2] == '4' ? 17 : 16;
        else if (e && e[0] == 'w' && e[1] == 'z') {
            const int sc = e[2] == 'p' ? 1 : e[2] == 's' ? 2 : e[2] == '3' ? 3 : 0;
            const bool roll = e[sc ? 3 : 2] == '2';
            variant = sc == 1 ? 9 : sc == 2 ? (roll ? 14 : 13) : sc == 3 ? 15 : (roll ? 12 : 11);
        }
        else if (e && e[0] == 'r' && e[1] == 'q') variant = e[2] == '8' ? 8 : 7;
        else if (e && e[0] == 'r' && e[1] == 'p') variant = e[2] == '1' ? (e[3] == '2' ? 6 : 5) : 4;
        else if (e && e[0] == 'r') variant = 0;
        else if (e && e[0] == 'p' && e[4] == '3') variant = 3;
        else if (e && e[0] == 'p') variant = 2;
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

// the wz kernels read the tangent in the kz slot order (kz_key); k_linearize writes it that way:
// 0 = not kz (fp64, other kernels), 1 = compact kz order (default), 2 = fixed 64-slot kz blocks (MPL_KZ_PAD=1;
// measured 9 % slower at cfg4)
// fp64 HVP (MPL_HVP_KERNEL64): "wh" (default: k_hvp_wh<double, 3>, one cell's 45 doubles per lane) or
// "sel" (the MPL_HVP_KERNEL selection, whose fp32-only variants fall back to k_hvp_rp<double, 10>)
int hvp_variant64() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPL_HVP_KERNEL64");
        v = (e && e[0] == 's') ? hvp_variant() : 18;
    }
    return v;
}
int hvp_kz_layout(int precision) {
    static int pad = -1;
    if (pad < 0) {
        const char *e = getenv("MPL_KZ_PAD");
        pad = (e && e[0] == '1') ? 1 : 0;
    }
    if (precision != 32) return hvp_variant64() == 18 ? 3 : 0;
    if (hvp_variant() == 16 || hvp_variant() == 17) return 3;  // wh: natural compact order (slot = rank)
    if (hvp_variant() < 9 || hvp_variant() > 15) return 0;
    return pad ? 2 : 1;
}

// Hu (tile-dense) must be zero on every node that receives atomics (all non-interior nodes).
template <class T>
mpl_status launch_hvp(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu, const CGSlot *cgs, int cgj,
                      double cgthr) {
    if (ctx->T == 0) return MPL_OK;
    int variant = hvp_variant();
    if (sizeof(T) == 8) {
        variant = hvp_variant64();
        if (variant == 16 || variant == 17 || variant == 18)
            return launch_wh<T, 3>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);  // 45 doubles per lane
    }
    if (variant == 16 || variant == 17) {
        if (sizeof(T) == 4)
            return variant == 16 ? launch_wh<T, 5>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr)
                                 : launch_wh<T, 4>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr);
        variant = 5;
    }
    if (variant >= 9 && variant <= 15) {
        if (sizeof(T) == 4) {
            const bool pad = hvp_kz_layout(32) == 2;
#define WZ(M, R, S) (pad ? launch_wz<M, R, S, true>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr) \
                         : launch_wz<M, R, S, false>(ctx, u_tile, Hu_tile, uHu, cgs, cgj, cgthr))
            if (variant == 9) return WZ(3, false, WZ_PLANE);
            if (variant == 11) return WZ(3, false, WZ_RMW);
            if (variant == 14) return WZ(2, true, WZ_SHFL);
            if (variant == 13) return WZ(3, false, WZ_SHFL);
            if (variant == 15) return WZ(3, false, WZ_RMW3);
            if (variant == 12) return WZ(2, true, WZ_RMW);
#undef WZ
        }
        variant = 5;
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
