// k_load.cu — SURVEY §8(a) row a9: Load (Alg. 4).
//   cells with m_c > 0: v_c = sum_i w_ic v_i (w_ic = 1/8), G_c = sum_i v_i (x) grad w_ic
//   particles: v_p = sum_c w_cp v_c, G_p = sum_c w_cp G_c (w at x_p^n)                   (Eqs. vc2p, Gc2p)
//              x_p += dt v_p ; F_p <- (I + dt G_p) F_p
// plus the quadrature/particle export helpers of the C ABI.
#include <cub/cub.cuh>

#include "mpl_common.cuh"

namespace {

__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

template <class T> __device__ __forceinline__ void st_vec12(T *dst, const T *v);
template <> __device__ __forceinline__ void st_vec12<float>(float *dst, const float *v) {
    float4 *d = reinterpret_cast<float4 *>(dst);
#pragma unroll
    for (int i = 0; i < 3; i++) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
template <> __device__ __forceinline__ void st_vec12<double>(double *dst, const double *v) {
    double2 *d = reinterpret_cast<double2 *>(dst);
#pragma unroll
    for (int i = 0; i < 6; i++) d[i] = make_double2(v[2 * i], v[2 * i + 1]);
}
template <class T> __device__ __forceinline__ void ld_vec12(const T *src, T *v);
template <> __device__ __forceinline__ void ld_vec12<float>(const float *src, float *v) {
    const float4 *s = reinterpret_cast<const float4 *>(src);
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const float4 x = __ldg(s + i);
        v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
    }
}
template <> __device__ __forceinline__ void ld_vec12<double>(const double *src, double *v) {
    const double2 *s = reinterpret_cast<const double2 *>(src);
#pragma unroll
    for (int i = 0; i < 6; i++) {
        const double2 x = __ldg(s + i);
        v[2 * i] = x.x; v[2 * i + 1] = x.y;
    }
}

// per cell: (v_c, G_c) from the 5^3 node halo, packed as 12 reals [v_c (3), G_c (9)] so G2P gathers a
// cell with three 16-byte loads (fp32)
template <class T>
__global__ void __launch_bounds__(128) k_n2c(GridP g, const int *__restrict__ nplus, const int *__restrict__ cstart,
                                             const uint8_t *__restrict__ clocal, const int *__restrict__ hascells,
                                             const T *__restrict__ q_m, const vec4<T> *__restrict__ v,
                                             T *__restrict__ vG) {
    __shared__ vec4<T> vh[125];
    const int t = blockIdx.x, tid = threadIdx.x;
    (void)hascells;  // every tile with structural cells: on a slab rank that includes the ghost plane
    const int cs = cstart[t], nc = cstart[t + 1] - cs;
    if (nc == 0) return;
    for (int h = tid; h < 125; h += blockDim.x) {
        int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        int dp = ((hx >> 2) << 2) | ((hy >> 2) << 1) | (hz >> 2);
        int tt = dp ? nplus[8 * t + dp] : t;
        vh[h] = tt >= 0 ? v[(int64_t)tt * 64 + local_id(hx & 3, hy & 3, hz & 3)] : mk4<T>(0, 0, 0, 0);
    }
    __syncthreads();
    if (tid >= nc) return;
    const int64_t cc = cs + tid;
    int l = clocal[cc];
    vec4<T> vv = mk4<T>(0, 0, 0, 0);
    T G[9];
#pragma unroll
    for (int a = 0; a < 9; a++) G[a] = T(0);
    if (l != 0xFF && q_m[cc] != T(0)) {
        int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
        const T q = T(0.25 * g.inv_dx);
#pragma unroll
        for (int o = 0; o < 8; o++) {
            int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            vec4<T> u = vh[((lx + ox) * 5 + ly + oy) * 5 + lz + oz];
            T s0 = ox ? q : -q, s1 = oy ? q : -q, s2 = oz ? q : -q;
            vv.x += T(0.125) * u.x; vv.y += T(0.125) * u.y; vv.z += T(0.125) * u.z;
            G[0] += u.x * s0; G[1] += u.x * s1; G[2] += u.x * s2;
            G[3] += u.y * s0; G[4] += u.y * s1; G[5] += u.y * s2;
            G[6] += u.z * s0; G[7] += u.z * s1; G[8] += u.z * s2;
        }
    }
    T out[12] = {vv.x, vv.y, vv.z, G[0], G[1], G[2], G[3], G[4], G[5], G[6], G[7], G[8]};
    st_vec12<T>(vG + 12 * cc, out);
}

// the per-particle part of G2P once v_p, G_p are interpolated: advect, update F (per material law), store
template <class T>
__device__ __forceinline__ void c2p_finish(int64_t p, int64_t p0, bool fast, T *sm, double dt_, const T xp[3],
                                           const T vp[3], const T Gp[9], const T Fp[9], T *__restrict__ x,
                                           T *__restrict__ v, T *__restrict__ F, T *__restrict__ G,
                                           const int *__restrict__ mat, const MatP &mp) {
    const T dt = T(dt_);
    T A[9], Fn[9];
#pragma unroll
    for (int a = 0; a < 9; a++) A[a] = dt * Gp[a] + ((a % 4 == 0) ? T(1) : T(0));
    const int mk = mat[p];
    if (mp.kind[mk] == 2) {
        // water particle: J^{n+1} = (1 + dt tr G_p) J^n, F_p = J^{1/3} I (J - 1 kept exact in
        // the product (1 + a)(1 + b) - 1 = a + b + a b)
        T H[9];
#pragma unroll
        for (int a = 0; a < 9; a++) H[a] = Fp[a] - ((a % 4 == 0) ? T(1) : T(0));
        const T jm1 = det_ipm1(H), da = dt * (Gp[0] + Gp[4] + Gp[8]);
        const T jn1 = jm1 + da + jm1 * da;
        const T s = T(1) + mexpm1(mlog1p(jn1) / T(3));
#pragma unroll
        for (int a = 0; a < 9; a++) Fn[a] = (a % 4 == 0) ? s : T(0);
    } else if (mp.sigy[mk] > 0.0) {
        // plastic particle: F_p^{n+1} = Z((I + dt G_p) F_p), the same von Mises
        // return map as the quadrature slots: F^E = F^tr + F^tr (P - I)
        T Ftr[9], H[9], Pm1[9], FP[9];
        mm3(A, Fp, Ftr);
#pragma unroll
        for (int a = 0; a < 9; a++) H[a] = Ftr[a] - ((a % 4 == 0) ? T(1) : T(0));
        vm_plastic_Pm1(H, T(mp.mu[mk]), T(mp.sigy[mk]), Pm1);
        mm3(Ftr, Pm1, FP);
#pragma unroll
        for (int a = 0; a < 9; a++) Fn[a] = Ftr[a] + FP[a];
    } else {
        mm3(A, Fp, Fn);
    }
    T xn[3];
#pragma unroll
    for (int a = 0; a < 3; a++) xn[a] = xp[a] + dt * vp[a];
    if (fast) {
        warp_store_aos<T, 3>(x, p0, sm, xn);
        warp_store_aos<T, 3>(v, p0, sm, vp);
        warp_store_aos<T, 9>(F, p0, sm, Fn);
        warp_store_aos<T, 9>(G, p0, sm, Gp);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
        x[3 * p + a] = xn[a];
        v[3 * p + a] = vp[a];
    }
#pragma unroll
    for (int a = 0; a < 9; a++) {
        F[9 * p + a] = Fn[a];
        G[9 * p + a] = Gp[a];
    }
}

// per particle (sorted order): interpolate, advect, update F
template <class T, int CMINB = 1>
__global__ void __launch_bounds__(256, CMINB) k_c2p(GridP g, double dt_, int64_t np, const int *__restrict__ skey, const int *__restrict__ pid,
                      const int *__restrict__ nplus,
                      const int *__restrict__ cellof, const T *__restrict__ vG,
                      T *__restrict__ x, T *__restrict__ v, T *__restrict__ F, T *__restrict__ G,
                      const int *__restrict__ mat, MatP mp) {
    // full warps without ghosts move x, F (in) and x, v, F, G (out) with 16-byte accesses through
    // shared memory; others per lane
    __shared__ __align__(16) T wsm[8][32 * 9];
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = p < np && pid[p] >= 0;  // ghosts (slab ranks) are advected by their owner
    const bool fast = __all_sync(0xffffffffu, valid);
    T *sm = wsm[threadIdx.x >> 5];
    const int64_t p0 = p & ~(int64_t)31;
    if (!valid) return;
    const int key = skey[p];
    const int t = key >> 6, l = key & 63;
    const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    T xp[3], f[3];
    if (fast) warp_load_aos<T, 3>(x, p0, sm, xp);
    else
#pragma unroll
        for (int a = 0; a < 3; a++) xp[a] = x[3 * p + a];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        T tt = (xp[a] - T(g.origin[a])) * T(g.inv_dx) - T(0.5);
        f[a] = tt - floor(tt);
    }
    T vp[3] = {0, 0, 0}, Gp[9];
#pragma unroll
    for (int a = 0; a < 9; a++) Gp[a] = T(0);
#pragma unroll
    for (int o = 0; o < 8; o++) {
        int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
        int cx = lx + ox, cy = ly + oy, cz = lz + oz;
        int dp = ((cx >> 2) << 2) | ((cy >> 2) << 1) | (cz >> 2);
        int tt = dp ? nplus[8 * t + dp] : t;
        int cc = cellof[tt * 64 + local_id(cx & 3, cy & 3, cz & 3)];
        T w = (ox ? f[0] : T(1) - f[0]) * (oy ? f[1] : T(1) - f[1]) * (oz ? f[2] : T(1) - f[2]);
        T c[12];
        ld_vec12<T>(vG + 12 * (int64_t)cc, c);
        vp[0] += w * c[0]; vp[1] += w * c[1]; vp[2] += w * c[2];
#pragma unroll
        for (int a = 0; a < 9; a++) Gp[a] += w * c[3 + a];
    }
    T Fp[9];
    if (fast) warp_load_aos<T, 9>(F, p0, sm, Fp);
    else
#pragma unroll
        for (int a = 0; a < 9; a++) Fp[a] = F[9 * p + a];
    c2p_finish<T>(p, p0, fast, sm, dt_, xp, vp, Gp, Fp, x, v, F, G, mat, mp);
}


// G2P per tile (default, MPL_G2P=tile): one CTA per tile stages the (v_c, G_c) of the 5^3 cells its
// particles' stencils reach in shared memory once (a per-particle gather looked up 8 cells through the
// neighbour table and the cell map: three dependent loads each), then its warps take the aligned
// 32-particle chunks of the tile's particle range [bstart[64 t], bstart[64 t + 64]) (particles are sorted
// by tile and base cell); chunks straddling a range end are processed lane by lane.
template <class T>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 8 : 4) k_c2p_tile(GridP g, double dt_, const int *__restrict__ bstart,
                                                  const int *__restrict__ skey, const int *__restrict__ pid,
                                                  const int *__restrict__ nplus, const int *__restrict__ cellof,
                                                  const T *__restrict__ vG, T *__restrict__ x, T *__restrict__ v,
                                                  T *__restrict__ F, T *__restrict__ G, const int *__restrict__ mat,
                                                  MatP mp) {
    __shared__ __align__(16) T cv[125 * 12];
    __shared__ __align__(16) T wsm[4][32 * 12];
    const int t = blockIdx.x, tid = threadIdx.x;
    const int pb = bstart[64 * t], pe = bstart[64 * t + 64];
    if (pb == pe) return;
    if (tid < 125) {
        const int X = tid / 25, Y = (tid / 5) % 5, Z = tid % 5;
        const int dp = ((X >> 2) << 2) | ((Y >> 2) << 1) | (Z >> 2);
        const int tt = dp ? nplus[8 * t + dp] : t;
        const int cc = tt < 0 ? -1 : cellof[tt * 64 + local_id(X & 3, Y & 3, Z & 3)];
        T c[12];
        if (cc >= 0) ld_vec12<T>(vG + 12 * (int64_t)cc, c);
        else
#pragma unroll
            for (int a = 0; a < 12; a++) c[a] = T(0);
        st_vec12<T>(cv + 12 * tid, c);
    }
    __syncthreads();
    const int w = tid >> 5, lane = tid & 31;
    T *sm = wsm[w];
    for (int64_t p0 = ((int64_t)pb & ~(int64_t)31) + 32 * w; p0 < pe; p0 += 128) {
        const int64_t p = p0 + lane;
        const bool valid = p >= pb && p < pe && pid[p] >= 0;  // ghosts (slab ranks) are advected by their owner
        const bool fast = __all_sync(0xffffffffu, valid);
        if (!valid) continue;
        const int l = skey[p] & 63;
        const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
        T xp[3], f[3], Fp[9];  // x and F requested together (one memory round trip per chunk)
        if (fast) {
            // the chunk's x (32 x 3) and F (32 x 9) as 16-byte vectors, all loads issued before any is used
            constexpr int NX = (int)(32 * 3 * sizeof(T) / 16), NF = (int)(32 * 9 * sizeof(T) / 16);
            constexpr int KX = (NX + 31) / 32, KF = (NF + 31) / 32;
            const float4 *sx = reinterpret_cast<const float4 *>(x + 3 * p0);
            const float4 *sF = reinterpret_cast<const float4 *>(F + 9 * p0);
            float4 rx[KX], rF[KF];
#pragma unroll
            for (int k = 0; k < KX; k++)
                if (lane + 32 * k < NX) rx[k] = sx[lane + 32 * k];
#pragma unroll
            for (int k = 0; k < KF; k++)
                if (lane + 32 * k < NF) rF[k] = sF[lane + 32 * k];
            float4 *dx4 = reinterpret_cast<float4 *>(sm), *dF4 = reinterpret_cast<float4 *>(sm + 32 * 3);
#pragma unroll
            for (int k = 0; k < KX; k++)
                if (lane + 32 * k < NX) dx4[lane + 32 * k] = rx[k];
#pragma unroll
            for (int k = 0; k < KF; k++)
                if (lane + 32 * k < NF) dF4[lane + 32 * k] = rF[k];
            __syncwarp();
#pragma unroll
            for (int a = 0; a < 3; a++) xp[a] = sm[lane * 3 + a];
#pragma unroll
            for (int a = 0; a < 9; a++) Fp[a] = sm[32 * 3 + lane * 9 + a];
            __syncwarp();
        } else {
#pragma unroll
            for (int a = 0; a < 3; a++) xp[a] = x[3 * p + a];
#pragma unroll
            for (int a = 0; a < 9; a++) Fp[a] = F[9 * p + a];
        }
#pragma unroll
        for (int a = 0; a < 3; a++) {
            T tt = (xp[a] - T(g.origin[a])) * T(g.inv_dx) - T(0.5);
            f[a] = tt - floor(tt);
        }
        T vp[3] = {0, 0, 0}, Gp[9];
#pragma unroll
        for (int a = 0; a < 9; a++) Gp[a] = T(0);
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            const T w8 = (ox ? f[0] : T(1) - f[0]) * (oy ? f[1] : T(1) - f[1]) * (oz ? f[2] : T(1) - f[2]);
            const T *c = cv + 12 * (((lx + ox) * 5 + ly + oy) * 5 + lz + oz);
            T cc[12];
            if (sizeof(T) == 4) {
                const float4 *c4 = reinterpret_cast<const float4 *>(c);
#pragma unroll
                for (int i = 0; i < 3; i++) {
                    const float4 q = c4[i];
                    cc[4 * i] = q.x; cc[4 * i + 1] = q.y; cc[4 * i + 2] = q.z; cc[4 * i + 3] = q.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 12; i++) cc[i] = c[i];
            }
            vp[0] += w8 * cc[0]; vp[1] += w8 * cc[1]; vp[2] += w8 * cc[2];
#pragma unroll
            for (int a = 0; a < 9; a++) Gp[a] += w8 * cc[3 + a];
        }
        c2p_finish<T>(p, p0, fast, sm, dt_, xp, vp, Gp, Fp, x, v, F, G, mat, mp);
    }
}

// sorted -> input order: out[id[p]] = in[p] (width w)
template <class T>
__global__ void k_unsort(int64_t np, int w, const int *__restrict__ id, const T *__restrict__ in, T *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= np * w) return;
    int64_t p = i / w;
    int a = (int)(i % w);
    out[(int64_t)id[p] * w + a] = in[i];
}

// quadrature export: tau, S from the slot data (S = I + E)
template <class T>
__global__ void k_export_q(int64_t C, int nmat, GridP g, const int *__restrict__ coord, const int *__restrict__ cstart,
                           int T_, const uint8_t *__restrict__ clocal, const int *__restrict__ ccanon,
                           const T *__restrict__ q_m, const T *__restrict__ q_mv, const T *__restrict__ q_mG,
                           const T *__restrict__ q_slot, int32_t *__restrict__ ijk, T *__restrict__ m_c,
                           T *__restrict__ v_c, T *__restrict__ G_c, T *__restrict__ V_ck, T *__restrict__ tau_ck,
                           T *__restrict__ S_ck, int64_t nout) {
    int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cc >= C) return;
    int o = ccanon[cc];
    if (o < 0) return;
    // find tile by binary search on cstart
    int lo = 0, hi = T_;
    while (hi - lo > 1) {
        int mid = (lo + hi) / 2;
        if (cstart[mid] <= cc) lo = mid; else hi = mid;
    }
    int l = clocal[cc];
    ijk[3 * o + 0] = coord[3 * lo] * 4 + (l >> 4);
    ijk[3 * o + 1] = coord[3 * lo + 1] * 4 + ((l >> 2) & 3);
    ijk[3 * o + 2] = coord[3 * lo + 2] * 4 + (l & 3);
    T m = q_m[cc];
    m_c[o] = m;
    T im = m != T(0) ? T(1) / m : T(0);
    for (int a = 0; a < 3; a++) v_c[3 * o + a] = q_mv[3 * cc + a] * im;
    for (int a = 0; a < 9; a++) G_c[9 * o + a] = q_mG[9 * cc + a] * im;
    const int sym[9] = {0, 3, 5, 3, 1, 4, 5, 4, 2};
    for (int k = 0; k < nmat; k++) {
        const T *sl = q_slot + (cc * nmat + k) * 16;
        V_ck[(int64_t)k * nout + o] = sl[0];
        for (int a = 0; a < 9; a++) {
            tau_ck[((int64_t)k * nout + o) * 9 + a] = sl[7 + sym[a]];
            S_ck[((int64_t)k * nout + o) * 9 + a] = sl[1 + sym[a]] + ((a % 4 == 0) ? T(1) : T(0));
        }
    }
}

// exported cells: structural cells of owned tiles (hascells), one thread per padded slot
__global__ void k_ccanon_flags(const int *__restrict__ cstart, const int *__restrict__ hascells,
                               const uint8_t *__restrict__ clocal, int *__restrict__ act) {
    const int t = blockIdx.x;
    const int cs = cstart[t], ce = cstart[t + 1];
    if (cs + (int)threadIdx.x < ce) act[cs + threadIdx.x] = hascells[t] && clocal[cs + threadIdx.x] != 0xFF;
}
__global__ void k_ccanon_fix(int64_t C, const int *__restrict__ act, int *__restrict__ canon) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < C && !act[i]) canon[i] = -1;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

template <class T>
mpl_status g2p_impl(mpl_ctx ctx, double dt) {
    cudaStream_t st = ctx->stream;
    const int T_ = ctx->T;
    const int c = ctx->cur;
    MPL_CHECK(ghost_nodes_from_upper<T>(ctx, ctx->n_v.p));  // slab ranks: next slab's second node plane
    if (T_)
        k_n2c<T><<<T_, 128, 0, st>>>(ctx->grid, (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p,
                                     (const uint8_t *)ctx->c_local.p, (const int *)ctx->t_hascells.p,
                                     (const T *)ctx->q_m.p, (const vec4<T> *)ctx->n_v.p, (T *)ctx->q_vc.p);
        ctx->launches++;
    static int g2p_tile = -1;
    if (g2p_tile < 0) {
        const char *e = getenv("MPL_G2P");
        g2p_tile = (e && e[0] == 'p') ? 0 : 1;  // "particle": one thread per particle with its own cell lookups
    }
    if (ctx->np && g2p_tile && T_) {
        k_c2p_tile<T><<<T_, 128, 0, st>>>(ctx->grid, dt, (const int *)ctx->t_bstart.p, (const int *)ctx->pskey.p,
                                          (const int *)ctx->pid[c].p, (const int *)ctx->t_nplus.p,
                                          (const int *)ctx->t_cellof.p, (const T *)ctx->q_vc.p, (T *)ctx->px[c].p,
                                          (T *)ctx->pv.p, (T *)ctx->pF[c].p, (T *)ctx->pG.p,
                                          (const int *)ctx->pmat[c].p, ctx->mats);
        ctx->launches++;
    } else if (ctx->np) {
        static int cmb = -1;
        if (cmb < 0) {
            const char *e = getenv("MPL_C2P_MINB");
            cmb = e ? atoi(e) : 4;  // 4 CTAs per SM (64 registers): cfg4 G2P 0.94 -> 0.82 ms, cfg3 PPC 64 4.48 -> 3.83
        }
        if (cmb == 4) k_c2p<T, 4><<<nblk(ctx->np, 256), 256, 0, st>>>(ctx->grid, dt, ctx->np, (const int *)ctx->pskey.p,
                                                    (const int *)ctx->pid[c].p,
                                                    (const int *)ctx->t_nplus.p, (const int *)ctx->t_cellof.p,
                                                    (const T *)ctx->q_vc.p,
                                                    (T *)ctx->px[c].p, (T *)ctx->pv.p, (T *)ctx->pF[c].p,
                                                    (T *)ctx->pG.p, (const int *)ctx->pmat[c].p,
                                                    ctx->mats);
        else k_c2p<T><<<nblk(ctx->np, 256), 256, 0, st>>>(ctx->grid, dt, ctx->np, (const int *)ctx->pskey.p,
                                                    (const int *)ctx->pid[c].p,
                                                    (const int *)ctx->t_nplus.p, (const int *)ctx->t_cellof.p,
                                                    (const T *)ctx->q_vc.p,
                                                    (T *)ctx->px[c].p, (T *)ctx->pv.p, (T *)ctx->pF[c].p,
                                                    (T *)ctx->pG.p, (const int *)ctx->pmat[c].p,
                                                    ctx->mats);
        ctx->launches++;
    }
    MPL_CUDA(cudaGetLastError());
    MPL_CUDA(cudaStreamSynchronize(st));
    ctx->vg_unsorted = false;  // k_c2p wrote v, G in the sorted order
    ctx->resampled = false;  // quadrature state is consumed
    ctx->linearized = false;
    ctx->solved = false;
    return MPL_OK;
}

template <class T>
mpl_status export_particles(mpl_ctx ctx, void *x, void *v, void *F, void *G) {
    if (multi(ctx)) return export_owned_particles<T>(ctx, x, v, F, G, nullptr, nullptr);
    MPL_CHECK(sync_vg_order<T>(ctx));
    cudaStream_t st = ctx->stream;
    const int64_t np = ctx->np;
    const int c = ctx->cur;
    MPL_CHECK(ensure(ctx, ctx->io_stage2, (size_t)(np * 9 + 16) * sizeof(T)));
    struct Item { void *dst; const void *src; int w; };
    Item items[4] = {{x, ctx->px[c].p, 3}, {v, ctx->pv.p, 3}, {F, ctx->pF[c].p, 9}, {G, ctx->pG.p, 9}};
    for (auto &it : items) {
        if (!it.dst || !np) continue;
        k_unsort<T><<<nblk(np * it.w, 256), 256, 0, st>>>(np, it.w, (const int *)ctx->pid[c].p, (const T *)it.src,
                                                          (T *)ctx->io_stage2.p); ctx->launches++;
        MPL_CUDA(cudaMemcpyAsync(it.dst, ctx->io_stage2.p, np * it.w * sizeof(T), cudaMemcpyDefault, st));
    }
    MPL_CUDA(cudaGetLastError());
    MPL_CUDA(cudaStreamSynchronize(st));
    return MPL_OK;
}

// Pipelined readback: unsort x, v, F, G into the readback set on the compute stream (after whatever
// step was enqueued last), then D2H on the copy stream; the next async readback waits until these
// copies have drained the readback set (ev_rb_done).  mpl_stage_wait synchronises the copy stream.
template <class T>
mpl_status export_particles_async(mpl_ctx ctx, void *x, void *v, void *F, void *G) {
    MPL_CHECK(io_streams(ctx));
    MPL_CHECK(sync_vg_order<T>(ctx));
    cudaStream_t st = ctx->stream, cs = ctx->rstream;
    const int64_t np = ctx->np;
    const int c = ctx->cur;
    if (ctx->rb_once) MPL_CUDA(cudaStreamWaitEvent(st, ctx->ev_rb_done, 0));
    struct Item { void *dst; const void *src; int w; };
    Item items[4] = {{x, ctx->px[c].p, 3}, {v, ctx->pv.p, 3}, {F, ctx->pF[c].p, 9}, {G, ctx->pG.p, 9}};
    for (int i = 0; i < 4; i++) {
        if (!items[i].dst || !np) continue;
        MPL_CUDA(cudaStreamSynchronize(cs));  // ensure() may reallocate rb[i]
        MPL_CHECK(ensure(ctx, ctx->rb[i], (size_t)np * items[i].w * sizeof(T)));
        k_unsort<T><<<nblk(np * items[i].w, 256), 256, 0, st>>>(np, items[i].w, (const int *)ctx->pid[c].p,
                                                                (const T *)items[i].src, (T *)ctx->rb[i].p);
        ctx->launches++;
    }
    MPL_CUDA(cudaGetLastError());
    MPL_CUDA(cudaEventRecord(ctx->ev_rb_ready, st));
    MPL_CUDA(cudaStreamWaitEvent(cs, ctx->ev_rb_ready, 0));
    for (int i = 0; i < 4; i++)
        if (items[i].dst && np)
            MPL_CUDA(cudaMemcpyAsync(items[i].dst, ctx->rb[i].p, np * items[i].w * sizeof(T), cudaMemcpyDefault, cs));
    MPL_CUDA(cudaEventRecord(ctx->ev_rb_done, cs));
    ctx->rb_once = true;
    return MPL_OK;
}

template mpl_status export_particles_async<float>(mpl_ctx, void *, void *, void *, void *);
template mpl_status export_particles_async<double>(mpl_ctx, void *, void *, void *, void *);

template <class T>
mpl_status export_quadrature(mpl_ctx ctx, int32_t *ijk, void *m_c, void *v_c, void *G_c, void *V_ck, void *tau_ck,
                             void *S_ck) {
    cudaStream_t st = ctx->stream;
    const int64_t C = ctx->C, n = ctx->n_cells_active;
    const int nm = ctx->mats.nmat;
    const size_t s = sizeof(T);
    // canonical cell index = rank among non-padding compact cells
    DevBuf act, canon, out;
    auto cleanup = [&]() {
        cudaFree(act.p);
        cudaFree(canon.p);
        cudaFree(out.p);
    };
    size_t nbytes_out = n * 3 * 4 + n * s * (1 + 3 + 9 + nm * (1 + 9 + 9)) + 256;
    if (cudaMalloc(&act.p, C * 4 + 16) != cudaSuccess || cudaMalloc(&canon.p, C * 4 + 16) != cudaSuccess ||
        cudaMalloc(&out.p, nbytes_out) != cudaSuccess) {
        cleanup();
        ctx->err = "out of device memory in export_quadrature";
        return MPL_ERR_OOM;
    }
    if (C) {
        k_ccanon_flags<<<ctx->T, 64, 0, st>>>((const int *)ctx->t_cstart.p, (const int *)ctx->t_hascells.p,
                                              (const uint8_t *)ctx->c_local.p, (int *)act.p); ctx->launches++;
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int *)act.p, (int *)canon.p, (int)C, st);
        void *tp = nullptr;
        cudaMalloc(&tp, tmp + 16);
        cub::DeviceScan::ExclusiveSum(tp, tmp, (const int *)act.p, (int *)canon.p, (int)C, st);
        k_ccanon_fix<<<nblk(C, 256), 256, 0, st>>>(C, (const int *)act.p, (int *)canon.p); ctx->launches++;
        char *o = (char *)out.p;
        int32_t *d_ijk = (int32_t *)o; o += n * 3 * 4;
        T *d_m = (T *)o; o += n * s;
        T *d_v = (T *)o; o += n * 3 * s;
        T *d_G = (T *)o; o += n * 9 * s;
        T *d_V = (T *)o; o += n * nm * s;
        T *d_tau = (T *)o; o += n * nm * 9 * s;
        T *d_S = (T *)o;
        k_export_q<T><<<nblk(C, 256), 256, 0, st>>>(C, nm, ctx->grid, (const int *)ctx->t_coord.p,
                                                    (const int *)ctx->t_cstart.p, ctx->T, (const uint8_t *)ctx->c_local.p,
                                                    (const int *)canon.p, (const T *)ctx->q_m.p, (const T *)ctx->q_mv.p,
                                                    (const T *)ctx->q_mG.p, (const T *)ctx->q_slot.p, d_ijk, d_m, d_v, d_G,
                                                    d_V, d_tau, d_S, n); ctx->launches++;
        if (ijk) cudaMemcpyAsync(ijk, d_ijk, n * 3 * 4, cudaMemcpyDefault, st);
        if (m_c) cudaMemcpyAsync(m_c, d_m, n * s, cudaMemcpyDefault, st);
        if (v_c) cudaMemcpyAsync(v_c, d_v, n * 3 * s, cudaMemcpyDefault, st);
        if (G_c) cudaMemcpyAsync(G_c, d_G, n * 9 * s, cudaMemcpyDefault, st);
        if (V_ck) cudaMemcpyAsync(V_ck, d_V, n * nm * s, cudaMemcpyDefault, st);
        if (tau_ck) cudaMemcpyAsync(tau_ck, d_tau, n * nm * 9 * s, cudaMemcpyDefault, st);
        if (S_ck) cudaMemcpyAsync(S_ck, d_S, n * nm * 9 * s, cudaMemcpyDefault, st);
        cudaStreamSynchronize(st);
        cudaFree(tp);
    }
    cudaError_t e = cudaGetLastError();
    cleanup();
    if (e != cudaSuccess) {
        ctx->err = std::string("CUDA error in export_quadrature: ") + cudaGetErrorString(e);
        return MPL_ERR_CUDA;
    }
    return MPL_OK;
}

template mpl_status g2p_impl<float>(mpl_ctx, double);
template mpl_status g2p_impl<double>(mpl_ctx, double);
template mpl_status export_particles<float>(mpl_ctx, void *, void *, void *, void *);
template mpl_status export_particles<double>(mpl_ctx, void *, void *, void *, void *);
template mpl_status export_quadrature<float>(mpl_ctx, int32_t *, void *, void *, void *, void *, void *, void *);
template mpl_status export_quadrature<double>(mpl_ctx, int32_t *, void *, void *, void *, void *, void *, void *);
