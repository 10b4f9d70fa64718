#include <algorithm>
// k_resample.cu — SURVEY §8(a) rows a0-a4: binning + activation, particle sort, P2Q scatter
// (as a race-free per-cell gather over base-cell buckets), stretch reconstruction, C2N gather.
//
// Paper: Alg. 2 Unload; Eqs. p2c-mV / p2c-mv-affine / p2c-A-sum;
// Eq. vtau; C2N; stretch bases Alg. 3 lines 4-7 with the
// StVK-Hencky closed form Eqs. hencky-trace / hencky-ei / hencky-sigmai.
#include <cub/cub.cuh>

#include "mpl_common.cuh"

namespace {

__device__ __forceinline__ int dense_id(const GridP &g, int bx, int by, int bz) {
    return (bx * g.nb[1] + by) * g.nb[2] + bz;
}
__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

// ---- a0: base cell, domain check, active cell blocks ------------------------------------------
template <class T>
__global__ void k_bin_flags(GridP g, int64_t np, const T *__restrict__ x, const int *__restrict__ pid,
                            int *__restrict__ base, int *__restrict__ cflag, DevScalars *sc) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned live = __ballot_sync(0xffffffffu, p < np);
    if (p >= np) return;
    int b[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        T t = (x[3 * p + a] - T(g.origin[a])) * T(g.inv_dx) - T(0.5);
        T fb = floor(t);
        b[a] = (int)fb;
        ok = ok && (fb >= T(0)) && (b[a] <= g.n[a] - 2) && (t == t);
    }
    const int key = (b[0] << 20) | (b[1] << 10) | b[2];
    // particles arrive sorted by base cell (the previous step's order): only the first lane of a run of
    // equal base cells flags the run's (1-8) cell blocks, with plain stores (no read of the flag)
    const unsigned ok_m = __ballot_sync(live, ok);
    const int prev = __shfl_up_sync(live, key, 1);
    if (!ok) {
        atomicMin(&sc->oob_particle, pid[p]);
        base[p] = -1;
        return;
    }
    base[p] = key;
    const int lane = threadIdx.x & 31;
    const bool first = lane == 0 || !((ok_m >> (lane - 1)) & 1u) || prev != key;
    if (!first) return;
    int b0[3] = {b[0] >> 2, b[1] >> 2, b[2] >> 2}, b1[3] = {(b[0] + 1) >> 2, (b[1] + 1) >> 2, (b[2] + 1) >> 2};
    for (int o = 0; o < 8; o++) {
        int bx = (o & 4) ? b1[0] : b0[0], by = (o & 2) ? b1[1] : b0[1], bz = (o & 1) ? b1[2] : b0[2];
        if (((o & 4) && b1[0] == b0[0]) || ((o & 2) && b1[1] == b0[1]) || ((o & 1) && b1[2] == b0[2])) continue;
        cflag[dense_id(g, bx, by, bz)] = 1;
    }
}

// active node blocks = cell blocks dilated by +{0,1}^3; also counts active cell blocks
__global__ void k_node_flags(GridP g, const int *__restrict__ cflag, int *__restrict__ nflag,
                             unsigned long long *nblocks, int xlo, int xhi) {
    int d = blockIdx.x * blockDim.x + threadIdx.x;
    int N = g.nb[0] * g.nb[1] * g.nb[2];
    if (d >= N || !cflag[d]) return;
    int bz = d % g.nb[2], by = (d / g.nb[2]) % g.nb[1], bx = d / (g.nb[1] * g.nb[2]);
    if (bx >= xlo && bx < xhi) atomicAdd(nblocks, 1ull);  // owned cell blocks (slab)
    for (int o = 0; o < 8; o++) {
        int x = bx + ((o >> 2) & 1), y = by + ((o >> 1) & 1), z = bz + (o & 1);
        if (x < g.nb[0] && y < g.nb[1] && z < g.nb[2]) nflag[dense_id(g, x, y, z)] = 1;
    }
}

// tile_of (exclusive scan of nflag) -> tile coords; tile_of[d] = -1 where inactive
__global__ void k_tiles(GridP g, const int *__restrict__ nflag, int *__restrict__ tile_of, int *__restrict__ coord) {
    int d = blockIdx.x * blockDim.x + threadIdx.x;
    int N = g.nb[0] * g.nb[1] * g.nb[2];
    if (d >= N) return;
    if (nflag[d]) {
        int t = tile_of[d];
        coord[3 * t + 0] = d / (g.nb[1] * g.nb[2]);
        coord[3 * t + 1] = (d / g.nb[2]) % g.nb[1];
        coord[3 * t + 2] = d % g.nb[2];
    } else {
        tile_of[d] = -1;
    }
}

// hascells[t]: the tile's cell block is active AND owned by this slab rank (physics runs on it);
// cell blocks outside the slab (ghost planes) keep their structural cells for P2Q / G2P only.
__global__ void k_tile_nbrs(GridP g, int T, const int *__restrict__ coord, const int *__restrict__ tile_of,
                            const int *__restrict__ cflag, int *__restrict__ nplus, int *__restrict__ nminus,
                            int *__restrict__ hascells, int xlo, int xhi) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    int c[3] = {coord[3 * t], coord[3 * t + 1], coord[3 * t + 2]};
    for (int o = 0; o < 8; o++) {
        int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
        int x = c[0] + ox, y = c[1] + oy, z = c[2] + oz;
        nplus[8 * t + o] = (x < g.nb[0] && y < g.nb[1] && z < g.nb[2]) ? tile_of[dense_id(g, x, y, z)] : -1;
        x = c[0] - ox; y = c[1] - oy; z = c[2] - oz;
        nminus[8 * t + o] = (x >= 0 && y >= 0 && z >= 0) ? tile_of[dense_id(g, x, y, z)] : -1;
    }
    hascells[t] = cflag[dense_id(g, c[0], c[1], c[2])] && c[0] >= xlo && c[0] < xhi;
}

// bucket key (tile*64 + local base cell) and rank inside the bucket
__global__ void k_count(GridP g, int64_t np, const int *__restrict__ base, const int *__restrict__ tile_of,
                        int *__restrict__ key, int *__restrict__ rank, int *__restrict__ bcount) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned act = __ballot_sync(0xffffffffu, p < np);
    if (p >= np) return;
    int b = base[p];
    int bx = b >> 20, by = (b >> 10) & 1023, bz = b & 1023;
    int t = tile_of[dense_id(g, bx >> 2, by >> 2, bz >> 2)];
    DASSERT(t >= 0 && b >= 0);
    int k = t * 64 + local_id(bx & 3, by & 3, bz & 3);
    key[p] = k;
    // warp-aggregated: the lanes of one bucket (particles arrive sorted by the previous step's buckets, so
    // runs are long at high PPC) take one atomic for the run and ranks in lane order
    const unsigned peers = __match_any_sync(act, k);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    int r0 = 0;
    if (lane == leader) r0 = atomicAdd(&bcount[k], __popc(peers));
    r0 = __shfl_sync(peers, r0, leader);
    rank[p] = r0 + __popc(peers & ((1u << lane) - 1u));
}

// ---- Kirchhoff stress of a particle, StVK-Hencky ------------------------
// tau = mu log b + lam/2 tr(log b) I with log b from eig(b - I), b - I = H + H^T + H H^T, H = F - I
template <class T>
__device__ __forceinline__ void hencky_tau(const T F[9], T mu, T lam, T tau[6]) {
    T H[9];
#pragma unroll
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? T(1) : T(0));
    T B[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            B[3 * a + b] = H[3 * a + b] + H[3 * b + a] + H[3 * a] * H[3 * b] + H[3 * a + 1] * H[3 * b + 1] +
                           H[3 * a + 2] * H[3 * b + 2];
    T w[3], Q[9];
    sym_eig3(B, w, Q);
    T l0 = mlog1p(w[0]), l1 = mlog1p(w[1]), l2 = mlog1p(w[2]);
    T tr = T(0.5) * lam * (l0 + l1 + l2);
    T t0 = mu * l0 + tr, t1 = mu * l1 + tr, t2 = mu * l2 + tr;
    // tau = Q diag(t) Q^T, packed xx yy zz xy yz xz
    tau[0] = Q[0] * Q[0] * t0 + Q[1] * Q[1] * t1 + Q[2] * Q[2] * t2;
    tau[1] = Q[3] * Q[3] * t0 + Q[4] * Q[4] * t1 + Q[5] * Q[5] * t2;
    tau[2] = Q[6] * Q[6] * t0 + Q[7] * Q[7] * t1 + Q[8] * Q[8] * t2;
    tau[3] = Q[0] * Q[3] * t0 + Q[1] * Q[4] * t1 + Q[2] * Q[5] * t2;
    tau[4] = Q[3] * Q[6] * t0 + Q[4] * Q[7] * t1 + Q[5] * Q[8] * t2;
    tau[5] = Q[0] * Q[6] * t0 + Q[1] * Q[7] * t1 + Q[2] * Q[8] * t2;
}

// ---- Kirchhoff stress of a particle, split Neo-Hookean (Eq. split-nh-tau), packed
template <class T>
__device__ __forceinline__ void nh_tau(const T F[9], T mu, T kappa, T tau[6]) {
    T H[9];
#pragma unroll
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? T(1) : T(0));
    T B[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            B[3 * a + b] = H[3 * a + b] + H[3 * b + a] + H[3 * a] * H[3 * b] + H[3 * a + 1] * H[3 * b + 1] +
                           H[3 * a + 2] * H[3 * b + 2];
    const T jm1 = det_ipm1(H);
    const T j23 = mexpm1(T(-2.0 / 3.0) * mlog1p(jm1));  // J^{-2/3} - 1
    const T trB3 = (B[0] + B[4] + B[8]) / T(3);
    const T s = mu * (T(1) + j23), al = T(0.5) * kappa * jm1 * (T(2) + jm1);
    tau[0] = s * (B[0] - trB3) + al;
    tau[1] = s * (B[4] - trB3) + al;
    tau[2] = s * (B[8] - trB3) + al;
    tau[3] = s * B[1];
    tau[4] = s * B[5];
    tau[5] = s * B[2];
}

// ---- J-based water (§4.5): tau = pi I, pi = kappa J (J - 1), J = det F_p ----------------
// (the particle carries only J; kappa = E).  J - 1 from the cancellation-free det(I + H) - 1.
template <class T>
__device__ __forceinline__ void water_tau(const T F[9], T kappa, T tau[6]) {
    T H[9];
#pragma unroll
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? T(1) : T(0));
    const T jm1 = det_ipm1(H);
    const T pi = kappa * (T(1) + jm1) * jm1;
    tau[0] = tau[1] = tau[2] = pi;
    tau[3] = tau[4] = tau[5] = T(0);
}

// Water slot base stretch (Eq. J_base) in fp64: pi_c = tr(tau_c)/3, r = 1 + 4 pi_c/kappa
// (clamped at 0), J_base - 1 = (r - 1) / (2 (sqrt r + 1)), S = J_base^{1/3} I -> E = (J_base^{1/3} - 1) I.
__device__ __forceinline__ void water_stretch_E(const double tau[6], double kappa, double E[6]) {
    const double x = 4.0 * (tau[0] + tau[1] + tau[2]) / (3.0 * kappa);  // r - 1
    const double xr = x < -1.0 ? -1.0 : x;
    const double jbm1 = xr / (2.0 * (sqrt(1.0 + xr) + 1.0));
    const double sm1 = expm1(log1p(jbm1) / 3.0);
    E[0] = E[1] = E[2] = sm1;
    E[3] = E[4] = E[5] = 0.0;
}

// ---- split Neo-Hookean stretch reconstruction (App. C), in fp64 -------
// tau = U diag(tau_i) U^T; alpha = tr/3; J = sqrt(1 + 2 alpha / kappa); s = mu J^{-2/3};
// delta_i = (tau_i - alpha)/s; m solves m^3 + S2 m + (S3 - J^2) = 0 on the branch m > -min delta
// (Cardano, Vieta form of the one-real-root case, Newton-polished); beta_i = m + delta_i;
// returns E = S - I = U diag(sqrt(beta_i) - 1) U^T.  false outside the inversion domain.
__device__ __forceinline__ double cbrt_s(double z) { return cbrt(z); }
__device__ bool nh_stretch_E(const double tau[6], double mu, double kappa, double E[6]) {
    double A[9] = {tau[0], tau[3], tau[5], tau[3], tau[1], tau[4], tau[5], tau[4], tau[2]};
    double w[3], U[9];
    sym_eig3(A, w, U);
    const double alpha = (w[0] + w[1] + w[2]) / 3.0;
    const double J2m1 = 2.0 * alpha / kappa;  // J^2 - 1
    if (!(J2m1 > -1.0)) return false;
    const double J2 = 1.0 + J2m1, J = sqrt(J2);
    const double s = mu * exp(-log1p(J2m1) / 3.0);  // mu J^{-2/3}
    double d[3];
    for (int i = 0; i < 3; i++) d[i] = (w[i] - alpha) / s;
    const double p = d[0] * d[1] + d[1] * d[2] + d[2] * d[0], q = d[0] * d[1] * d[2] - J2;
    const double dmin = fmin(d[0], fmin(d[1], d[2]));
    const double D = 0.25 * q * q + p * p * p / 27.0;
    double m;
    if (D >= 0.0) {
        const double u = cbrt_s(-0.5 * q + (q <= 0.0 ? sqrt(D) : -sqrt(D)));
        m = u != 0.0 ? u - p / (3.0 * u) : 0.0;
    } else {
        const double r = 2.0 * sqrt(-p / 3.0);
        double arg = (1.5 * q / p) * sqrt(-3.0 / p);
        arg = fmin(1.0, fmax(-1.0, arg));
        const double th = acos(arg) / 3.0;
        m = -1e300;
        for (int k = 0; k < 3; k++) {
            const double mk = r * cos(th - 2.0943951023931953 * k);
            if (mk > -dmin && mk > m) m = mk;
        }
    }
    for (int it = 0; it < 3; it++) {  // Newton polish on the same cubic
        const double f = m * m * m + p * m + q, df = 3.0 * m * m + p;
        if (!(fabs(df) > 1e-300)) break;
        const double mn = m - f / df;
        if (!(mn > -dmin)) break;
        m = mn;
    }
    double em[3];
    for (int i = 0; i < 3; i++) {
        const double beta = m + d[i];
        if (!(beta > 0.0)) return false;
        em[i] = (beta - 1.0) / (sqrt(beta) + 1.0);  // sigma_i - 1
    }
    E[0] = U[0] * U[0] * em[0] + U[1] * U[1] * em[1] + U[2] * U[2] * em[2];
    E[1] = U[3] * U[3] * em[0] + U[4] * U[4] * em[1] + U[5] * U[5] * em[2];
    E[2] = U[6] * U[6] * em[0] + U[7] * U[7] * em[1] + U[8] * U[8] * em[2];
    E[3] = U[0] * U[3] * em[0] + U[1] * U[4] * em[1] + U[2] * U[5] * em[2];
    E[4] = U[3] * U[6] * em[0] + U[4] * U[7] * em[1] + U[5] * U[8] * em[2];
    E[5] = U[0] * U[6] * em[0] + U[1] * U[7] * em[1] + U[2] * U[8] * em[2];
    return true;
}

// ---- particle scatter into sorted order + P2Q record ------------------------------------------
// record (24 reals): f(3) fraction in the base cell, m_p, a = m_p (v_p - dx G_p f) (3),
// m_p G_p (9), V_p, V_p tau_p (6), material id (as real)
constexpr int REC = 24;
template <class T> __device__ __forceinline__ void st_rec(T *dst, const T *r);
template <> __device__ __forceinline__ void st_rec<float>(float *dst, const float *r) {
    float4 *d4 = reinterpret_cast<float4 *>(dst);
#pragma unroll
    for (int i = 0; i < REC / 4; i++) d4[i] = make_float4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
}
template <> __device__ __forceinline__ void st_rec<double>(double *dst, const double *r) {
    double2 *d2 = reinterpret_cast<double2 *>(dst);
#pragma unroll
    for (int i = 0; i < REC / 2; i++) d2[i] = make_double2(r[2 * i], r[2 * i + 1]);
}
template <class T>
__global__ void k_scatter(GridP g, MatP mp, int64_t np, const int *__restrict__ key, const int *__restrict__ rank,
                          const int *__restrict__ bstart, const T *__restrict__ x, const T *__restrict__ v,
                          const T *__restrict__ F, const T *__restrict__ G, const T *__restrict__ vol,
                          const int *__restrict__ mat, const int *__restrict__ pid, T *__restrict__ xo,
                          T *__restrict__ Fo, T *__restrict__ volo, int *__restrict__ mato, int *__restrict__ pido,
                          int *__restrict__ keyo, T *__restrict__ rec, DevScalars *sc) {
    // full warps load x, v, F, G with 16-byte accesses through shared memory, others per lane
    __shared__ __align__(16) T wsm[8][32 * 9];
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool fast = __all_sync(0xffffffffu, p < np);
    T xp[3], vp[3], Fp[9], Gp[9];
    if (fast) {
        T *sm = wsm[threadIdx.x >> 5];
        const int64_t p0 = p & ~(int64_t)31;
        warp_load_aos<T, 3>(x, p0, sm, xp);
        warp_load_aos<T, 3>(v, p0, sm, vp);
        warp_load_aos<T, 9>(F, p0, sm, Fp);
        warp_load_aos<T, 9>(G, p0, sm, Gp);
    }
    if (p >= np) return;
    if (!fast) {
#pragma unroll
        for (int a = 0; a < 3; a++) { xp[a] = x[3 * p + a]; vp[a] = v[3 * p + a]; }
#pragma unroll
        for (int a = 0; a < 9; a++) { Fp[a] = F[9 * p + a]; Gp[a] = G[9 * p + a]; }
    }
    int k = key[p];
    int64_t d = bstart[k] + rank[p];
    DASSERT(k >= 0 && d >= 0 && d < np);
    T Vp = vol[p];
    int m = mat[p];
    int id = pid[p];
    if (det3(Fp) <= T(0)) atomicMin(&sc->inv_particle, id);
    T mu = T(mp.mu[m]), lam = T(mp.lam[m]);
    T mass = T(mp.rho[m]) * Vp;
    T tau[6];
    if (mp.kind[m] == 1) nh_tau(Fp, mu, T(mp.kappa[m]), tau);  // Alg. 2 line 3, per-material law
    else if (mp.kind[m] == 2) water_tau(Fp, T(mp.kappa[m]), tau);
    else hencky_tau(Fp, mu, lam, tau);
    T f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        T t = (xp[a] - T(g.origin[a])) * T(g.inv_dx) - T(0.5);
        f[a] = t - floor(t);
    }
    T dx = T(g.dx);
    T r[REC];  // assembled in registers, written with 16-byte stores (the destination is scattered)
    r[0] = f[0]; r[1] = f[1]; r[2] = f[2];
    r[3] = mass;
#pragma unroll
    for (int a = 0; a < 3; a++) r[4 + a] = mass * (vp[a] - dx * (Gp[3 * a] * f[0] + Gp[3 * a + 1] * f[1] + Gp[3 * a + 2] * f[2]));
#pragma unroll
    for (int a = 0; a < 9; a++) r[7 + a] = mass * Gp[a];
    r[16] = Vp;
#pragma unroll
    for (int a = 0; a < 6; a++) r[17 + a] = Vp * tau[a];
    r[23] = T(m);
    st_rec<T>(rec + d * REC, r);
#pragma unroll
    for (int a = 0; a < 3; a++) xo[3 * d + a] = xp[a];
#pragma unroll
    for (int a = 0; a < 9; a++) Fo[9 * d + a] = Fp[a];
    volo[d] = Vp;
    mato[d] = m;
    pido[d] = id;
    keyo[d] = k;
}

// ---- the sort as a gather (MPL_SORT=gather, default): src[d] = p for the destination d of particle p,
// then destination-ordered threads read their source particle (per-particle contiguous AoS, scattered
// reads) and write the sorted state and the P2Q record in destination order: whole warps store
// contiguous 16-byte vectors (warp_store_aos) instead of 32 scattered scalar stores per field
__global__ void k_sort_src(int64_t np, const int *__restrict__ key, const int *__restrict__ rank,
                           const int *__restrict__ bstart, int *__restrict__ src) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < np) src[bstart[key[p]] + rank[p]] = (int)p;
}

template <class T>
__global__ void __launch_bounds__(256) k_scatter_g(GridP g, MatP mp, int64_t np, const int *__restrict__ src,
                                                   const int *__restrict__ key, const T *__restrict__ x,
                                                   const T *__restrict__ v, const T *__restrict__ F,
                                                   const T *__restrict__ G, const T *__restrict__ vol,
                                                   const int *__restrict__ mat, const int *__restrict__ pid,
                                                   T *__restrict__ xo, T *__restrict__ Fo, T *__restrict__ volo,
                                                   int *__restrict__ mato, int *__restrict__ pido,
                                                   int *__restrict__ keyo, T *__restrict__ rec, DevScalars *sc) {
    __shared__ __align__(16) T wsm[8][32 * REC];
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool fast = __all_sync(0xffffffffu, d < np);
    if (!fast && d >= np) return;
    const int p = src[d];
    DASSERT(p >= 0 && p < np);
    T xp[3], vp[3], Fp[9], Gp[9];
#pragma unroll
    for (int a = 0; a < 3; a++) { xp[a] = x[3 * (int64_t)p + a]; vp[a] = v[3 * (int64_t)p + a]; }
#pragma unroll
    for (int a = 0; a < 9; a++) { Fp[a] = F[9 * (int64_t)p + a]; Gp[a] = G[9 * (int64_t)p + a]; }
    const int k = key[p];
    const T Vp = vol[p];
    const int m = mat[p];
    const int id = pid[p];
    if (det3(Fp) <= T(0)) atomicMin(&sc->inv_particle, id);
    const T mu = T(mp.mu[m]), lam = T(mp.lam[m]);
    const T mass = T(mp.rho[m]) * Vp;
    T tau[6];
    if (mp.kind[m] == 1) nh_tau(Fp, mu, T(mp.kappa[m]), tau);  // Alg. 2 line 3, per-material law
    else if (mp.kind[m] == 2) water_tau(Fp, T(mp.kappa[m]), tau);
    else hencky_tau(Fp, mu, lam, tau);
    T f[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const T t = (xp[a] - T(g.origin[a])) * T(g.inv_dx) - T(0.5);
        f[a] = t - floor(t);
    }
    const T dx = T(g.dx);
    T r[REC];
    r[0] = f[0]; r[1] = f[1]; r[2] = f[2];
    r[3] = mass;
#pragma unroll
    for (int a = 0; a < 3; a++) r[4 + a] = mass * (vp[a] - dx * (Gp[3 * a] * f[0] + Gp[3 * a + 1] * f[1] + Gp[3 * a + 2] * f[2]));
#pragma unroll
    for (int a = 0; a < 9; a++) r[7 + a] = mass * Gp[a];
    r[16] = Vp;
#pragma unroll
    for (int a = 0; a < 6; a++) r[17 + a] = Vp * tau[a];
    r[23] = T(m);
    volo[d] = Vp;
    mato[d] = m;
    pido[d] = id;
    keyo[d] = k;
    if (fast) {
        T *sm = wsm[threadIdx.x >> 5];
        const int64_t d0 = d & ~(int64_t)31;
        warp_store_aos<T, REC>(rec, d0, sm, r);
        warp_store_aos<T, 3>(xo, d0, sm, xp);
        warp_store_aos<T, 9>(Fo, d0, sm, Fp);
    } else {
        st_rec<T>(rec + d * REC, r);
#pragma unroll
        for (int a = 0; a < 3; a++) xo[3 * d + a] = xp[a];
#pragma unroll
        for (int a = 0; a < 9; a++) Fo[9 * d + a] = Fp[a];
    }
}

// v / G into the sorted order of the last k_scatter (see mpl_ctx_s::vg_unsorted)
template <class T>
__global__ void k_vg_to_sorted(int64_t np, const int *__restrict__ key, const int *__restrict__ rank,
                               const int *__restrict__ bstart, const T *__restrict__ v, const T *__restrict__ G,
                               T *__restrict__ vo, T *__restrict__ Go) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np) return;
    const int64_t d = bstart[key[p]] + rank[p];
#pragma unroll
    for (int a = 0; a < 3; a++) vo[3 * d + a] = v[3 * p + a];
#pragma unroll
    for (int a = 0; a < 9; a++) Go[9 * d + a] = G[9 * p + a];
}

// ---- structural cell masks: cell active iff some base-cell bucket in cell - {0,1}^3 is non-empty
__global__ void k_cell_mask(GridP g, int T_, const int *__restrict__ coord, const int *__restrict__ nminus,
                            const int *__restrict__ bcount, const int *__restrict__ hascells,
                            unsigned long long *__restrict__ cmask, int *__restrict__ ccount, int *__restrict__ ncell,
                            int *__restrict__ kcnt, unsigned long long *ncells, int *__restrict__ kcnt2) {
    int t = blockIdx.x;
    int l = threadIdx.x;  // 64 threads
    int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    int cx = coord[3 * t] * 4 + lx, cy = coord[3 * t + 1] * 4 + ly, cz = coord[3 * t + 2] * 4 + lz;
    bool act = false;
    if (cx < g.n[0] && cy < g.n[1] && cz < g.n[2]) {
        for (int o = 0; o < 8 && !act; o++) {
            int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            int bx = lx - ox, by = ly - oy, bz = lz - oz;
            if (cx - ox < 0 || cy - oy < 0 || cz - oz < 0) continue;
            int dm = ((bx < 0) << 2) | ((by < 0) << 1) | (bz < 0);
            int tt = nminus[8 * t + dm];
            if (tt < 0) continue;
            if (bcount[tt * 64 + local_id(bx & 3, by & 3, bz & 3)] > 0) act = true;
        }
    }
    unsigned int lo = __ballot_sync(0xffffffffu, act);
    __shared__ unsigned int part[2], pairs;
    if (l == 0) pairs = 0u;
    if ((l & 31) == 0) part[l >> 5] = lo;
    __syncthreads();
    // k_hvp_wz lanes holding a cell (kz_key(l) & 31 = the lane of cell l): the pair slots of the
    // compressed tangent layout, 2 KC_REALS reals each
    if (act) atomicOr(&pairs, 1u << (kz_key(l) & 31));
    __syncthreads();
    if (l == 0) {
        unsigned long long m = (unsigned long long)part[0] | ((unsigned long long)part[1] << 32);
        cmask[t] = m;
        int c = __popcll(m);
        ccount[t] = (c + 3) & ~3;
        ncell[t] = c;
        // tangent only on owned tiles: room for the full (45 c reals) or the compressed (2 KC_REALS per
        // pair slot) layout, rounded up to 4
        const int np = __popc(pairs);
        kcnt[t] = hascells[t] ? (45 * c + 3) & ~3 : 0;  // the 45-number layout
        kcnt2[t] = hascells[t] ? 2 * KC_REALS * np : 0;  // the compressed layout (its own offsets)
        if (c && hascells[t]) atomicAdd(ncells, (unsigned long long)c);
    }
}

// perm[t][j]: local position of the tile's j-th cell (j < n, increasing l), then its unoccupied
// positions in increasing order: a permutation of 0..63 that gives every HVP lane a distinct position.
__global__ void k_cell_list(int T_, const unsigned long long *__restrict__ cmask, const int *__restrict__ cstart,
                            uint8_t *__restrict__ clocal, int *__restrict__ cellof, uint8_t *__restrict__ perm) {
    int t = blockIdx.x;
    int l = threadIdx.x;
    unsigned long long m = cmask[t];
    int cs = cstart[t], ce = cstart[t + 1];
    int c = __popcll(m);
    const int r = __popcll(m & ((1ull << l) - 1ull));
    if ((m >> l) & 1ull) {
        clocal[cs + r] = (uint8_t)l;
        cellof[t * 64 + l] = cs + r;
        perm[t * 64 + r] = (uint8_t)l;
    } else {
        cellof[t * 64 + l] = -1;
        perm[t * 64 + c + (l - r)] = (uint8_t)l;
    }
    if (cs + c + l < ce) clocal[cs + c + l] = 0xFF;
}

template <class T> __device__ __forceinline__ void ld_rec(const T *__restrict__ src, T *r);
template <> __device__ __forceinline__ void ld_rec<float>(const float *__restrict__ src, float *r) {
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
#pragma unroll
    for (int i = 0; i < REC / 4; i++) {
        const float4 v = __ldg(s4 + i);
        r[4 * i] = v.x; r[4 * i + 1] = v.y; r[4 * i + 2] = v.z; r[4 * i + 3] = v.w;
    }
}
template <> __device__ __forceinline__ void ld_rec<double>(const double *__restrict__ src, double *r) {
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
#pragma unroll
    for (int i = 0; i < REC / 2; i++) {
        const double2 v = __ldg(s2 + i);
        r[2 * i] = v.x; r[2 * i + 1] = v.y;
    }
}

// ---- a2-a4, parallel form (default): 8 lanes per cell --------------------------------------------
// Lane o of a cell's 8-lane group gathers the base-cell bucket c - o (the particles whose stencil
// corner o is this cell); the 8 partial sums are combined with shuffles inside the aligned group;
// lane k then reconstructs material slot k's stretch (Eqs. hencky-ei/sigmai, or the split
// Neo-Hookean inversion) — the slots of a cell in parallel.  256 threads = half a tile (32 cells).
template <class T>
__device__ __forceinline__ T grp_sum(T v) {  // sum over the aligned 8-lane group
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    return v;
}

template <class T>
__device__ __forceinline__ void stretch_slot(const MatP &mp, int k, const T tau[6], T E[6], DevScalars *sc) {
    if (mp.kind[k] == 2) {
        double td[6], Ed[6];
#pragma unroll
        for (int a = 0; a < 6; a++) td[a] = (double)tau[a];
        water_stretch_E(td, mp.kappa[k], Ed);
#pragma unroll
        for (int a = 0; a < 6; a++) E[a] = T(Ed[a]);
        return;
    }
    if (mp.kind[k] == 1) {
        double td[6], Ed[6];
#pragma unroll
        for (int a = 0; a < 6; a++) td[a] = (double)tau[a];
        if (nh_stretch_E(td, mp.mu[k], mp.kappa[k], Ed)) {
#pragma unroll
            for (int a = 0; a < 6; a++) E[a] = T(Ed[a]);
        } else {
#pragma unroll
            for (int a = 0; a < 6; a++) E[a] = T(0);
            sc->nonfinite = 1;  // outside the inversion domain (reported by resample)
        }
        return;
    }
    const T mu = T(mp.mu[k]), lam = T(mp.lam[k]);
    T A[9] = {tau[0], tau[3], tau[5], tau[3], tau[1], tau[4], tau[5], tau[4], tau[2]};
    T w[3], U[9];
    sym_eig3(A, w, U);
    const T s = (w[0] + w[1] + w[2]) / (T(2) * mu + T(3) * lam);  // Eq. hencky-trace
    T em[3];
#pragma unroll
    for (int i = 0; i < 3; i++) em[i] = mexpm1((w[i] - lam * s) / (T(2) * mu));  // sigma_i - 1
    E[0] = U[0] * U[0] * em[0] + U[1] * U[1] * em[1] + U[2] * U[2] * em[2];
    E[1] = U[3] * U[3] * em[0] + U[4] * U[4] * em[1] + U[5] * U[5] * em[2];
    E[2] = U[6] * U[6] * em[0] + U[7] * U[7] * em[1] + U[8] * U[8] * em[2];
    E[3] = U[0] * U[3] * em[0] + U[1] * U[4] * em[1] + U[2] * U[5] * em[2];
    E[4] = U[3] * U[6] * em[0] + U[4] * U[7] * em[1] + U[5] * U[8] * em[2];
    E[5] = U[0] * U[6] * em[0] + U[1] * U[7] * em[1] + U[2] * U[8] * em[2];
}

// 3 CTAs per SM pinned: the kernel waits on its record loads (ncu: long scoreboard 75 %), and at
// 88 registers ptxas dropped it to 2 CTAs (cfg4 P2Q +0.4 ms); 4 CTAs (64 registers, spills) is no faster
template <class T, int NM>  // NM >= mp.nmat: register arrays sized for NM material slots
__global__ void __launch_bounds__(256, 3) k_p2q8(GridP g, MatP mp, const int *__restrict__ coord,
                                              const int *__restrict__ nminus, const int *__restrict__ bstart,
                                              const int *__restrict__ cellof, const T *__restrict__ rec,
                                              T *__restrict__ q_m, T *__restrict__ q_mv, T *__restrict__ q_mG,
                                              T *__restrict__ q_slot, T *__restrict__ q_Sp, DevScalars *sc) {
    const int t = blockIdx.x >> 1;
    const int l = ((blockIdx.x & 1) << 5) | (threadIdx.x >> 3), o = threadIdx.x & 7;
    const int cc = cellof[t * 64 + l];
    const int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    const int cx = coord[3 * t] * 4 + lx, cy = coord[3 * t + 1] * 4 + ly, cz = coord[3 * t + 2] * 4 + lz;
    const int nmat = mp.nmat;
    const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
    T m = 0, mv[3] = {0, 0, 0}, mG[9];
#pragma unroll
    for (int a = 0; a < 9; a++) mG[a] = 0;
    T V[NM], Vt[NM][6];
#pragma unroll
    for (int k = 0; k < NM; k++) {
        V[k] = 0;
#pragma unroll
        for (int a = 0; a < 6; a++) Vt[k][a] = 0;
    }
    if (cc >= 0 && cx - ox >= 0 && cy - oy >= 0 && cz - oz >= 0) {
        const int bx = lx - ox, by = ly - oy, bz = lz - oz;
        const int dm = ((bx < 0) << 2) | ((by < 0) << 1) | (bz < 0);
        const int tt = nminus[8 * t + dm];
        if (tt >= 0) {
            const int kk = tt * 64 + local_id(bx & 3, by & 3, bz & 3);
            const int s0 = bstart[kk], e0 = bstart[kk + 1];
            const T dx = T(g.dx);
#pragma unroll 2
            for (int p = s0; p < e0; p++) {
                // the 96-byte (fp32) record in 16-byte loads (a scalar load per field costs one L1
                // wavefront per lane: the 8 lanes of a group read 8 different buckets)
                T r[REC];
                ld_rec<T>(rec + (int64_t)p * REC, r);
                // cell = base + o  =>  w = prod_a (o_a ? f_a : 1 - f_a)
                const T w = (ox ? r[0] : T(1) - r[0]) * (oy ? r[1] : T(1) - r[1]) * (oz ? r[2] : T(1) - r[2]);
                m += w * r[3];
                // m (v + G (x_c - x_p)) = a + dx (mG) o   (x_c - x_p = dx (o - f))
                mv[0] += w * (r[4] + dx * ((ox ? r[7] : T(0)) + (oy ? r[8] : T(0)) + (oz ? r[9] : T(0))));
                mv[1] += w * (r[5] + dx * ((ox ? r[10] : T(0)) + (oy ? r[11] : T(0)) + (oz ? r[12] : T(0))));
                mv[2] += w * (r[6] + dx * ((ox ? r[13] : T(0)) + (oy ? r[14] : T(0)) + (oz ? r[15] : T(0))));
#pragma unroll
                for (int a = 0; a < 9; a++) mG[a] += w * r[7 + a];
                const int k = (int)r[23];
#pragma unroll
                for (int q = 0; q < NM; q++) {
                    if (q == k) {
                        V[q] += w * r[16];
#pragma unroll
                        for (int a = 0; a < 6; a++) Vt[q][a] += w * r[17 + a];
                    }
                }
            }
        }
    }
    // combine the 8 source buckets of the cell (inactive groups carry zeros and write nothing)
    m = grp_sum(m);
#pragma unroll
    for (int a = 0; a < 3; a++) mv[a] = grp_sum(mv[a]);
#pragma unroll
    for (int a = 0; a < 9; a++) mG[a] = grp_sum(mG[a]);
#pragma unroll
    for (int q = 0; q < NM; q++) {
        if (q >= nmat) break;  // uniform
        V[q] = grp_sum(V[q]);
#pragma unroll
        for (int a = 0; a < 6; a++) Vt[q][a] = grp_sum(Vt[q][a]);
    }
    if (cc < 0) return;
    if (o == 0) {
        q_m[cc] = m;
#pragma unroll
        for (int a = 0; a < 3; a++) q_mv[3 * (int64_t)cc + a] = mv[a];
    }
    if (o == 1)
#pragma unroll
        for (int a = 0; a < 9; a++) q_mG[9 * (int64_t)cc + a] = mG[a];
    // material slot k on lane k (nmat <= 8)
#pragma unroll
    for (int q = 0; q < NM; q++) {
        if (q != o || q >= nmat) continue;
        T *sl = q_slot + ((int64_t)cc * nmat + q) * 16;
        T tau[6] = {0, 0, 0, 0, 0, 0}, E[6] = {0, 0, 0, 0, 0, 0};
        if (V[q] != T(0)) {
            const T iv = T(1) / V[q];
#pragma unroll
            for (int a = 0; a < 6; a++) tau[a] = Vt[q][a] * iv;  // Eq. vtau normalisation
            stretch_slot<T>(mp, q, tau, E, sc);
        }
        sl[0] = V[q];
#pragma unroll
        for (int a = 0; a < 6; a++) { sl[1 + a] = E[a]; sl[7 + a] = tau[a]; }
        sl[13] = sl[14] = sl[15] = T(0);
        if (q_Sp) {  // plastic runs: the iterate's base starts at S_base (general 3x3 storage)
            T *sp = q_Sp + ((int64_t)cc * nmat + q) * 9;
            sp[0] = E[0]; sp[4] = E[1]; sp[8] = E[2];
            sp[1] = sp[3] = E[3];
            sp[5] = sp[7] = E[4];
            sp[2] = sp[6] = E[5];
        }
    }
}

// ---- a2, scatter form (MPL_P2Q=scatter): one CTA per tile, shared-memory accumulation -----------------
// The north_star's P2Q: the tile's particles (its base-cell buckets, contiguous after the counting sort)
// are staged in shared memory with coalesced 16-byte loads, each record read from DRAM once; thread
// (bucket b, corner o) sums the bucket's contributions to cell b + o (Eqs. p2c-mV, p2c-mv-affine,
// p2c-A-sum, vtau; the weight of corner o from the fraction f) and adds them into a 5^3-cell
// shared accumulator (the 8 threads of a bucket read the same records: shared-memory broadcasts); then
// the 27 cells all of whose source buckets lie in the tile are stored and the other 98 are added with
// global atomics into zeroed accumulators (neighbouring tiles contribute there).  k_p2q_finish then
// normalises tau = (V tau) / V and reconstructs the stretch per slot (a4).
// ---- bulk copy (TMA, cp.async.bulk) into shared memory completing on an mbarrier ----------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// P2Q flush (both scatter kernels): compact cell ids of the tile's 5^3 accumulator cells, then interior
// cells (local 1..3 on every axis) stored, the rest added.  Thread c < 125 of each half-CTA owns cell c: the
// first half writes m, mv, mG (13 values), the second the material slots (7 per slot), every destination
// offset a compile-time constant of the unrolled loops.  PV: value v of cell c = the sum over its (up to
// 8) source pairs (bucket c - o, corner o) at acc[v * 8 * 68 + 68 o + bucket]; else acc[c * NV + v].
// Needs 256 threads; ends the kernel (no barrier after it).
template <class T, int NM, bool PV>
__device__ __forceinline__ void p2q_flush(int t, int tid, int nmat, const int *__restrict__ nplus,
                                          const int *__restrict__ cellof, const T *acc, T *__restrict__ q_m,
                                          T *__restrict__ q_mv, T *__restrict__ q_mG, T *__restrict__ q_slot) {
    constexpr int NV = 13 + 7 * NM, PV_ROW = 8 * 68;
    __shared__ int ccs[125];
    if (tid < 125) {
        const int X = tid / 25, Y = (tid / 5) % 5, Z = tid % 5;
        const int dp = ((X >> 2) << 2) | ((Y >> 2) << 1) | (Z >> 2);
        const int tt = dp ? nplus[8 * t + dp] : t;
        ccs[tid] = tt < 0 ? -1 : cellof[tt * 64 + local_id(X & 3, Y & 3, Z & 3)];
    }
    __syncthreads();
    const int c = tid & 127, half = tid >> 7;
    if (c < 125 && ccs[c] >= 0) {
        const int64_t cc = ccs[c];
        const int X = c / 25, Y = (c / 5) % 5, Z = c % 5;
        const bool interior = X >= 1 && X <= 3 && Y >= 1 && Y <= 3 && Z >= 1 && Z <= 3;
        int src[8];
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int bx = X - ((o >> 2) & 1), by = Y - ((o >> 1) & 1), bz = Z - (o & 1);
            src[o] = (bx >= 0 && bx < 4 && by >= 0 && by < 4 && bz >= 0 && bz < 4) ? o * 68 + (bx * 16 + by * 4 + bz) : -1;
        }
        auto val = [&](int v) -> T {
            if constexpr (PV) {
                T sum = T(0);
#pragma unroll
                for (int o = 0; o < 8; o++)
                    if (src[o] >= 0) sum += acc[v * PV_ROW + src[o]];
                return sum;
            } else {
                return acc[c * NV + v];
            }
        };
        auto put = [&](T *dst, T x) {
            if (interior) *dst = x;
            else if (x != T(0)) atomicAdd(dst, x);
        };
        if (half == 0) {
            put(q_m + cc, val(0));
#pragma unroll
            for (int k = 0; k < 3; k++) put(q_mv + 3 * cc + k, val(1 + k));
#pragma unroll
            for (int k = 0; k < 9; k++) put(q_mG + 9 * cc + k, val(4 + k));
        } else {
#pragma unroll
            for (int q = 0; q < NM; q++) {
                if (q >= nmat) break;  // slots past the context's materials (NM is an upper bound)
                T *sl = q_slot + (cc * nmat + q) * 16;
                put(sl, val(13 + 7 * q));
#pragma unroll
                for (int k = 0; k < 6; k++) put(sl + 7 + k, val(14 + 7 * q + k));
            }
        }
    }
}

constexpr int P2Q_CAP = 256;  // particles staged per pass, double-buffered (2 x 24 KB of fp32 records)
template <int NM> struct P2QNV { static constexpr int V = 13 + 7 * NM; };  // m, mv 3, mG 9, per slot V + V tau 6
template <class T, int NM>
__global__ void __launch_bounds__(256) k_p2q_tile(GridP g, MatP mp, const int *__restrict__ coord,
                                                  const int *__restrict__ nplus, const int *__restrict__ bstart,
                                                  const int *__restrict__ cellof, const T *__restrict__ rec,
                                                  T *__restrict__ q_m, T *__restrict__ q_mv, T *__restrict__ q_mG,
                                                  T *__restrict__ q_slot) {
    constexpr int NV = P2QNV<NM>::V;
    extern __shared__ __align__(16) unsigned char p2q_smem[];
    T *acc = reinterpret_cast<T *>(p2q_smem);             // [125][NV]
    T *Rb = acc + ((125 * NV + 3) & ~3);                  // [2][P2Q_CAP][REC]: the staged passes
    __shared__ int bs[65];
    __shared__ __align__(8) uint64_t bar[2];
    const int t = blockIdx.x, tid = threadIdx.x;
    if (tid < 65) bs[tid] = bstart[t * 64 + tid];
    // PV: the pair sums go to private shared slots after the last pass (no shared atomics: sm_100 has no
    // native shared fp32 add, atomicAdd there is a CAS loop), reusing the accumulator + record space
    constexpr int PV_ROW = 8 * 68;  // value-major rows of 8 corner columns of 68 (64 buckets + pad)
    constexpr bool PV = (size_t)NV * PV_ROW * sizeof(T) <=
                        (size_t)((125 * NV + 3) & ~3) * sizeof(T) + (size_t)2 * P2Q_CAP * REC * sizeof(T);
    if (!PV)
        for (int i = tid; i < 125 * NV; i += blockDim.x) acc[i] = T(0);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int p0 = bs[0], p1 = bs[64];
    DASSERT(p1 >= p0);
    if (p0 == p1) return;  // no particles based in this tile (every thread sees the same)
    const int nmat = mp.nmat;
    const T dx = T(g.dx);
    // thread tid owns the (bucket, corner) pairs tid and tid + 256 (256 threads) and sums them over every
    // staged pass in registers; each pair is added into the shared accumulator once per tile
    struct Acc {
        T m, mv[3], mG[9], V[NM], Vt[NM][6];
    };
    Acc A2[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        A2[h].m = 0;
#pragma unroll
        for (int a = 0; a < 3; a++) A2[h].mv[a] = 0;
#pragma unroll
        for (int a = 0; a < 9; a++) A2[h].mG[a] = 0;
#pragma unroll
        for (int k = 0; k < NM; k++) {
            A2[h].V[k] = 0;
#pragma unroll
            for (int a = 0; a < 6; a++) A2[h].Vt[k][a] = 0;
        }
    }
    // the records of pass k (particles [p0 + k CAP, ...)) arrive in buffer k & 1 by one bulk copy (TMA),
    // issued a pass ahead so it overlaps the previous pass's arithmetic
    auto issue = [&](int k) {
        const int c0 = p0 + k * P2Q_CAP, cn = min(P2Q_CAP, p1 - c0);
        const uint32_t bytes = (uint32_t)(cn * REC * sizeof(T));
        mbar_expect_tx(&bar[k & 1], bytes);
        bulk_g2s(Rb + (k & 1) * P2Q_CAP * REC, rec + (int64_t)c0 * REC, bytes, &bar[k & 1]);
    };
    const int npass = (p1 - p0 + P2Q_CAP - 1) / P2Q_CAP;
    if (tid == 0) issue(0);
    for (int k = 0; k < npass; k++) {
        const int c0 = p0 + k * P2Q_CAP, cn = min(P2Q_CAP, p1 - c0);
        if (tid == 0 && k + 1 < npass) issue(k + 1);  // buffer (k + 1) & 1 was released by the last barrier
        mbar_wait(&bar[k & 1], (uint32_t)((k >> 1) & 1));
        const T *R = Rb + (k & 1) * P2Q_CAP * REC;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int pr = tid + 256 * h;
            const int b = pr >> 3, o = pr & 7;
            const int s0 = max(bs[b], c0), e0 = min(bs[b + 1], c0 + cn);
            const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            Acc &q_ = A2[h];
            for (int p = s0; p < e0; p++) {
                T r[REC];  // the staged record, 16-byte shared loads
                {
                    const float4 *r4 = reinterpret_cast<const float4 *>(R + (p - c0) * REC);
                    float4 *d4 = reinterpret_cast<float4 *>(r);
#pragma unroll
                    for (int i = 0; i < (int)(REC * sizeof(T) / 16); i++) d4[i] = r4[i];
                }
                const T w = (ox ? r[0] : T(1) - r[0]) * (oy ? r[1] : T(1) - r[1]) * (oz ? r[2] : T(1) - r[2]);
                q_.m += w * r[3];
                // the affine term dx (mG)_p o of Eq. p2c-mv-affine is added after the loop from the mG sum
                // (sum_p w m G_p o = (sum_p w m G_p) o): only the o-independent part here
                q_.mv[0] += w * r[4];
                q_.mv[1] += w * r[5];
                q_.mv[2] += w * r[6];
#pragma unroll
                for (int a = 0; a < 9; a++) q_.mG[a] += w * r[7 + a];
                const int k = (int)r[23];
#pragma unroll
                for (int qq = 0; qq < NM; qq++)
                    if (qq == k) {
                        q_.V[qq] += w * r[16];
#pragma unroll
                        for (int a = 0; a < 6; a++) q_.Vt[qq][a] += w * r[17 + a];
                    }
            }
        }
        __syncthreads();  // buffer k & 1 consumed before pass k + 2 refills it
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {  // sum_p w m (v_p + G_p (x_c - x_p)) = sum_p w a_p + dx (sum_p w m G_p) o
        const int o = (tid + 256 * h) & 7;
        const T ox = T((o >> 2) & 1), oy = T((o >> 1) & 1), oz = T(o & 1);
        Acc &q_ = A2[h];
#pragma unroll
        for (int a = 0; a < 3; a++)
            q_.mv[a] += dx * (ox * q_.mG[3 * a] + oy * q_.mG[3 * a + 1] + oz * q_.mG[3 * a + 2]);
    }
    if constexpr (PV) {
        // pair (b, o) -> column 68 o + b of every value row: a warp's 32 pairs (4 buckets x 8 corners) hit
        // 32 distinct banks (4 o + b mod 32), and the flush's reads of one corner over consecutive cells too
        T *P = acc;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int pr = tid + 256 * h;
            T *col = P + (pr & 7) * 68 + (pr >> 3);
            const Acc &q_ = A2[h];
            col[0] = q_.m;
#pragma unroll
            for (int a = 0; a < 3; a++) col[(1 + a) * PV_ROW] = q_.mv[a];
#pragma unroll
            for (int a = 0; a < 9; a++) col[(4 + a) * PV_ROW] = q_.mG[a];
#pragma unroll
            for (int qq = 0; qq < NM; qq++) {
                col[(13 + 7 * qq) * PV_ROW] = q_.V[qq];
#pragma unroll
                for (int a = 0; a < 6; a++) col[(14 + 7 * qq + a) * PV_ROW] = q_.Vt[qq][a];
            }
        }
    } else {
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int pr = tid + 256 * h;
        const int b = pr >> 3, o = pr & 7;
        if (bs[b] == bs[b + 1]) continue;  // empty bucket
        const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
        const int bx = b >> 4, by = (b >> 2) & 3, bz = b & 3;
        T *ac = acc + (((bx + ox) * 5 + by + oy) * 5 + bz + oz) * NV;
        const Acc &q_ = A2[h];
        atomicAdd(ac, q_.m);
#pragma unroll
        for (int a = 0; a < 3; a++) atomicAdd(ac + 1 + a, q_.mv[a]);
#pragma unroll
        for (int a = 0; a < 9; a++) atomicAdd(ac + 4 + a, q_.mG[a]);
#pragma unroll
        for (int qq = 0; qq < NM; qq++) {  // slots past nmat hold zeros (material ids are < nmat)
            atomicAdd(ac + 13 + 7 * qq, q_.V[qq]);
#pragma unroll
            for (int a = 0; a < 6; a++) atomicAdd(ac + 14 + 7 * qq + a, q_.Vt[qq][a]);
        }
    }
    }
    p2q_flush<T, NM, PV>(t, tid, nmat, nplus, cellof, acc, q_m, q_mv, q_mG, q_slot);
}

// ---- a2, scatter form for dense particle buckets (MPL_P2Q_HI, mean >= P2Q_HI_PPC particles per occupied
// base cell, e.g. cfg3 at PPC 27 / 64): in k_p2q_tile a staged pass of 256 consecutive particles covers only
// a few buckets when buckets hold tens of particles, so most (bucket, corner) threads idle.  Here warp w
// owns buckets 8w .. 8w + 7 (contiguous records) and walks them one at a time with all 32 lanes: lane
// (slot j, corner o) = 8 j + o sums corner o over the bucket's particles j, j + 4, ...; the records arrive
// in 32-record chunks cp.async double-buffered per warp; the 4 slot sums are combined by shuffles and the
// (bucket, corner) sum is written to the private slot of the same layout as k_p2q_tile's, then the same
// flush.  No CTA barrier inside the particle loop.
__device__ __forceinline__ void cp_async16_g2s(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait_() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
constexpr double P2Q_HI_PPC = 40.0;  // cfg3: PPC 64 (61 per cell) 11.4 -> 9.4 ms; PPC 27 (26 per cell) 4.86 -> 5.05 ms
template <class T, int NM>
__global__ void __launch_bounds__(256) k_p2q_hi(GridP g, MatP mp, const int *__restrict__ coord,
                                                const int *__restrict__ nplus, const int *__restrict__ bstart,
                                                const int *__restrict__ cellof, const T *__restrict__ rec,
                                                T *__restrict__ q_m, T *__restrict__ q_mv, T *__restrict__ q_mG,
                                                T *__restrict__ q_slot) {
    constexpr int NV = P2QNV<NM>::V, PV_ROW = 8 * 68;
    extern __shared__ __align__(16) unsigned char p2q_smem[];
    T *P = reinterpret_cast<T *>(p2q_smem);  // [NV][PV_ROW] pair sums
    T *stg = P + NV * PV_ROW;                  // [8 warps][2][32 REC] record chunks
    __shared__ int bs[65];
    const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid < 65) bs[tid] = bstart[t * 64 + tid];
    __syncthreads();
    if (bs[0] == bs[64]) return;  // no particles based in this tile (every thread sees the same)
    const int nmat = mp.nmat;
    const T dx = T(g.dx);
    const int o = lane & 7, j = lane >> 3;
    const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
    T *S = stg + w * 2 * 32 * REC;
    constexpr int NC = (int)(REC * sizeof(T) / 16);  // 16-byte pieces per record
    for (int bb = 0; bb < 8; bb++) {
        const int b = 8 * w + bb;
        const int s0 = bs[b], e0 = bs[b + 1];
        T m = 0, mv[3] = {0, 0, 0}, mG[9], V[NM], Vt[NM][6];
#pragma unroll
        for (int a = 0; a < 9; a++) mG[a] = 0;
#pragma unroll
        for (int k = 0; k < NM; k++) {
            V[k] = 0;
#pragma unroll
            for (int a = 0; a < 6; a++) Vt[k][a] = 0;
        }
        const int nch = (e0 - s0 + 31) >> 5;
        auto issue = [&](int k) {  // lane i: record s0 + 32 k + i
            const int p = s0 + 32 * k + lane;
            if (p < e0) {
                const char *src = reinterpret_cast<const char *>(rec + (int64_t)p * REC);
                char *dst = reinterpret_cast<char *>(S + ((k & 1) * 32 + lane) * REC);
#pragma unroll
                for (int i = 0; i < NC; i++) cp_async16_g2s(dst + 16 * i, src + 16 * i);
            }
            cp_async_commit_();
        };
        if (nch > 0) issue(0);
        for (int k = 0; k < nch; k++) {
            if (k + 1 < nch) {
                issue(k + 1);  // buffer (k + 1) & 1 was released by the __syncwarp closing chunk k - 1
                cp_async_wait_<1>();
            } else {
                cp_async_wait_<0>();
            }
            __syncwarp();
            const T *R = S + (k & 1) * 32 * REC;
            const int n = min(32, e0 - s0 - 32 * k);
            for (int q = j; q < n; q += 4) {
                T r[REC];
                {
                    const float4 *r4 = reinterpret_cast<const float4 *>(R + q * REC);
                    float4 *d4 = reinterpret_cast<float4 *>(r);
#pragma unroll
                    for (int i = 0; i < NC; i++) d4[i] = r4[i];
                }
                const T wt = (ox ? r[0] : T(1) - r[0]) * (oy ? r[1] : T(1) - r[1]) * (oz ? r[2] : T(1) - r[2]);
                m += wt * r[3];
#pragma unroll
                for (int a = 0; a < 3; a++) mv[a] += wt * r[4 + a];  // affine term below, from the mG sum
#pragma unroll
                for (int a = 0; a < 9; a++) mG[a] += wt * r[7 + a];
                const int km = (int)r[23];
#pragma unroll
                for (int qq = 0; qq < NM; qq++)
                    if (qq == km || NM == 1) {
                        V[qq] += wt * r[16];
#pragma unroll
                        for (int a = 0; a < 6; a++) Vt[qq][a] += wt * r[17 + a];
                    }
            }
            __syncwarp();  // chunk consumed before it is refilled
        }
        // combine the 4 slots of each corner (lanes o, o + 8, o + 16, o + 24); slot 0 writes the pair
        auto red = [&](T x) {
            x += __shfl_xor_sync(0xffffffffu, x, 8);
            x += __shfl_xor_sync(0xffffffffu, x, 16);
            return x;
        };
        m = red(m);
#pragma unroll
        for (int a = 0; a < 3; a++) mv[a] = red(mv[a]);
#pragma unroll
        for (int a = 0; a < 9; a++) mG[a] = red(mG[a]);
#pragma unroll
        for (int qq = 0; qq < NM; qq++) {
            V[qq] = red(V[qq]);
#pragma unroll
            for (int a = 0; a < 6; a++) Vt[qq][a] = red(Vt[qq][a]);
        }
        if (j == 0) {
            // sum_p w m (v_p + G_p (x_c - x_p)) = sum_p w a_p + dx (sum_p w m G_p) o
#pragma unroll
            for (int a = 0; a < 3; a++)
                mv[a] += dx * (T(ox) * mG[3 * a] + T(oy) * mG[3 * a + 1] + T(oz) * mG[3 * a + 2]);
            T *col = P + o * 68 + b;
            col[0] = m;
#pragma unroll
            for (int a = 0; a < 3; a++) col[(1 + a) * PV_ROW] = mv[a];
#pragma unroll
            for (int a = 0; a < 9; a++) col[(4 + a) * PV_ROW] = mG[a];
#pragma unroll
            for (int qq = 0; qq < NM; qq++) {
                col[(13 + 7 * qq) * PV_ROW] = V[qq];
#pragma unroll
                for (int a = 0; a < 6; a++) col[(14 + 7 * qq + a) * PV_ROW] = Vt[qq][a];
            }
        }
    }
    p2q_flush<T, NM, true>(t, tid, nmat, nplus, cellof, P, q_m, q_mv, q_mG, q_slot);
}

// cells with two or more occupied material slots (the compressed tangent covers one slot per cell)
// and cells with an occupied slot whose stretch base is not I (E = S - I != 0): the compressed tangent's
// PSD projection is exact only at S = I
template <class T>
__global__ void k_multislot(int64_t C, int nmat, const uint8_t *__restrict__ clocal, const T *__restrict__ q_slot,
                            unsigned long long *count, unsigned long long *nonid) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int k = 0;
    bool ni = false;
    if (c < C && clocal[c] != 0xFF)
        for (int q = 0; q < nmat; q++) {
            const T *sl = q_slot + (c * nmat + q) * 16;
            if (sl[0] != T(0)) {
                k++;
#pragma unroll
                for (int a = 1; a < 7; a++) ni = ni || sl[a] != T(0);
            }
        }
    const unsigned int b = __ballot_sync(0xffffffffu, k >= 2), bn = __ballot_sync(0xffffffffu, ni);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (unsigned long long)__popc(b));
    if ((threadIdx.x & 31) == 0 && bn) atomicAdd(nonid, (unsigned long long)__popc(bn));
}

// a4 after the scatter: per (cell, slot) tau = (V tau) / V (Eq. vtau) and the stretch base
template <class T>
__global__ void k_p2q_finish(int64_t C, MatP mp, const uint8_t *__restrict__ clocal, T *__restrict__ q_slot,
                             T *__restrict__ q_Sp, DevScalars *sc) {
    const int nmat = mp.nmat;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= C * nmat) return;
    const int64_t cc = i / nmat;
    const int q = (int)(i - cc * nmat);
    T *sl = q_slot + i * 16;
    T tau[6] = {0, 0, 0, 0, 0, 0}, E[6] = {0, 0, 0, 0, 0, 0};
    const T V0 = sl[0];
    const T V = clocal[cc] != 0xFF ? V0 : T(0);
    if (V != T(0)) {
        const T iv = T(1) / V;
#pragma unroll
        for (int a = 0; a < 6; a++) tau[a] = sl[7 + a] * iv;
        stretch_slot<T>(mp, q, tau, E, sc);
    }
    // an empty slot of a local cell is all zeros already (zeroed accumulators, P2Q adds nothing): only
    // occupied slots and non-local cells are written (sl[1..6] of an occupied slot held zeros, 13..15 stay 0)
    if (V != T(0) || V0 != T(0)) {
        sl[0] = V;
#pragma unroll
        for (int a = 0; a < 6; a++) { sl[1 + a] = E[a]; sl[7 + a] = tau[a]; }
        sl[13] = sl[14] = sl[15] = T(0);
    }
    if (q_Sp) {
        T *sp = q_Sp + i * 9;
        sp[0] = E[0]; sp[4] = E[1]; sp[8] = E[2];
        sp[1] = sp[3] = E[3];
        sp[5] = sp[7] = E[4];
        sp[2] = sp[6] = E[5];
    }
}

// ---- a3: C2N gather (Alg. 2 lines 16-22) + Newton target and Dirichlet sets ----------
// PH 0: gather + finish in one pass (one rank).  PH 1: gather only, n_vn = ((mv)_i, m_i) partial
// sums over this rank's cells (slab ranks; completed by c2n_halo).  PH 2: finish from n_vn.
// Only owned cells (hascells of their tile) contribute; own[i] marks the copy counted by this rank.
template <class T, int PH>
__global__ void __launch_bounds__(64) k_c2n(GridP g, BoxP bx, double dt, double gx, double gy, double gz,
                                            const int *__restrict__ coord, const int *__restrict__ nminus,
                                            const int *__restrict__ cellof, const int *__restrict__ hascells,
                                            const T *__restrict__ q_m, const T *__restrict__ q_mv,
                                            const T *__restrict__ q_mG, T *__restrict__ n_mass,
                                            uint8_t *__restrict__ n_flag, vec4<T> *__restrict__ n_vn,
                                            vec4<T> *__restrict__ n_vhat, vec4<T> *__restrict__ n_v,
                                            uint8_t *__restrict__ n_own, T *__restrict__ n_mown,
                                            unsigned long long *__restrict__ nfree) {
    int t = blockIdx.x;
    int l = threadIdx.x;
    int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
    int ix = coord[3 * t] * 4 + lx, iy = coord[3 * t + 1] * 4 + ly, iz = coord[3 * t + 2] * 4 + lz;
    int64_t nidx = (int64_t)t * 64 + l;
    T m = 0, mv[3] = {0, 0, 0};
    if (PH != 2) {
        const T hdx = T(0.5 * g.dx);
        for (int o = 0; o < 8; o++) {
            int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            int cx = ix - ox, cy = iy - oy, cz = iz - oz;  // node = cell + o
            if (cx < 0 || cy < 0 || cz < 0 || cx >= g.n[0] || cy >= g.n[1] || cz >= g.n[2]) continue;
            int bx_ = lx - ox, by_ = ly - oy, bz_ = lz - oz;
            int dm = ((bx_ < 0) << 2) | ((by_ < 0) << 1) | (bz_ < 0);
            int tt = nminus[8 * t + dm];
            if (tt < 0 || !hascells[tt]) continue;
            int cc = cellof[tt * 64 + local_id(bx_ & 3, by_ & 3, bz_ & 3)];
            if (cc < 0) continue;
            T mc = q_m[cc];
            if (mc == T(0)) continue;
            // x_i - x_c = dx (o - 1/2)
            T d0 = ox ? hdx : -hdx, d1 = oy ? hdx : -hdx, d2 = oz ? hdx : -hdx;
            const T *G = q_mG + 9 * (int64_t)cc;
            m += T(0.125) * mc;
            mv[0] += T(0.125) * (q_mv[3 * (int64_t)cc + 0] + G[0] * d0 + G[1] * d1 + G[2] * d2);
            mv[1] += T(0.125) * (q_mv[3 * (int64_t)cc + 1] + G[3] * d0 + G[4] * d1 + G[5] * d2);
            mv[2] += T(0.125) * (q_mv[3 * (int64_t)cc + 2] + G[6] * d0 + G[7] * d1 + G[8] * d2);
        }
        if (PH == 1) {
            n_vn[nidx] = mk4<T>(mv[0], mv[1], mv[2], m);
            n_own[nidx] = 1;
            return;
        }
    } else {
        vec4<T> a = n_vn[nidx];
        mv[0] = a.x; mv[1] = a.y; mv[2] = a.z; m = a.w;
    }
    vec4<T> vn = mk4<T>(0, 0, 0, 0), vh = mk4<T>(0, 0, 0, 0), v0 = mk4<T>(0, 0, 0, 0);
    uint8_t flag = 0, own = 0;
    if (m > T(0)) {
        T im = T(1) / m;
        vn = mk4<T>(mv[0] * im, mv[1] * im, mv[2] * im, 0);
        vh = mk4<T>(vn.x + T(dt * gx), vn.y + T(dt * gy), vn.z + T(dt * gz), m);
        flag = 1;
        own = PH == 2 ? n_own[nidx] : 1;
        v0 = mk4<T>(vh.x, vh.y, vh.z, 0);
        double xi[3] = {g.origin[0] + g.dx * ix, g.origin[1] + g.dx * iy, g.origin[2] + g.dx * iz};
        for (int b = 0; b < bx.nbox; b++) {
            bool in = true;
#pragma unroll
            for (int a = 0; a < 3; a++) in = in && (xi[a] >= bx.lo[b][a]) && (xi[a] <= bx.hi[b][a]);
            if (in) {
                flag |= 2;
                v0 = mk4<T>(T(bx.vel[b][0]), T(bx.vel[b][1]), T(bx.vel[b][2]), 0);
                break;
            }
        }
    }
    unsigned int fb = __ballot_sync(0xffffffffu, flag == 1 && own);
    if ((threadIdx.x & 31) == 0 && fb) atomicAdd(nfree, (unsigned long long)__popc(fb));
    n_mass[nidx] = m;
    n_flag[nidx] = flag;
    n_vn[nidx] = vn;
    n_vhat[nidx] = vh;
    n_v[nidx] = v0;
    n_own[nidx] = own;
    if (PH == 2) n_mown[nidx] = own ? m : T(0);
}

__global__ void k_node_active(int64_t N, const uint8_t *__restrict__ flag, int *__restrict__ act) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) act[i] = flag[i] & 1;
}
__global__ void k_node_canon(int64_t N, const uint8_t *__restrict__ flag, int *__restrict__ canon,
                             int *__restrict__ list) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    if (flag[i] & 1) {
        list[canon[i]] = (int)i;
    } else {
        canon[i] = -1;
    }
}

__global__ void k_iota(int64_t n, int *a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// particle sort (MPL_SORT): "gather" (k_sort_src + k_scatter_g, destination-ordered writes) or
// "scatter" (k_scatter, source-ordered threads storing at the destinations)
bool sort_gather() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPL_SORT");
        v = (e && e[0] == 's') ? 0 : 1;
    }
    return v == 1;
}

// P2Q form (MPL_P2Q): "scatter" (default: k_p2q_tile + k_p2q_finish) or "gather" (k_p2q8, 8 lanes per cell)
bool p2q_scatter() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPL_P2Q");
        v = (e && e[0] == 'g') ? 0 : 1;  // scatter default: cfg4 resample 4.15 vs 4.96 ms, cfg3 PPC 64 15.4 vs 21.1
    }
    return v == 1;
}

template <class I>
mpl_status exclusive_scan(mpl_ctx ctx, const I *in, I *out, int64_t n) {
    size_t tmp = 0;
    MPL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, ctx->stream));
    MPL_CHECK(ensure(ctx, ctx->scan_tmp, tmp + 256));
    MPL_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scan_tmp.p, tmp, in, out, (int)n, ctx->stream));
    ctx->launches += 2;  // cub: init + scan kernels
    return MPL_OK;
}

}  // namespace

// =============================================================================================
// host orchestration
// =============================================================================================
template <class T>
mpl_status import_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F, const void *G,
                            const void *vol, const int32_t *mat) {
    ctx->np = n;
    ctx->np_own = n;
    ctx->cur = 0;
    ctx->vg_unsorted = false;
    size_t s = sizeof(T);
    MPL_CHECK(ensure(ctx, ctx->px[0], n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->px[1], n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->pF[0], n * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->pF[1], n * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->pv, n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->pG, n * 9 * s));
    for (int i = 0; i < 2; i++) {
        MPL_CHECK(ensure(ctx, ctx->pvol[i], n * s));
        MPL_CHECK(ensure(ctx, ctx->pmat[i], n * 4));
        MPL_CHECK(ensure(ctx, ctx->pid[i], n * 4));
    }
    MPL_CHECK(ensure(ctx, ctx->pkey, n * 4));
    MPL_CHECK(ensure(ctx, ctx->prank, n * 4));
    MPL_CHECK(ensure(ctx, ctx->pbase, n * 4));
    MPL_CHECK(ensure(ctx, ctx->prec, n * REC * s));
    cudaStream_t st = ctx->stream;
    MPL_CUDA(cudaMemcpyAsync(ctx->px[0].p, x, n * 3 * s, cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemcpyAsync(ctx->pv.p, v, n * 3 * s, cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemcpyAsync(ctx->pF[0].p, F, n * 9 * s, cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemcpyAsync(ctx->pG.p, G, n * 9 * s, cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemcpyAsync(ctx->pvol[0].p, vol, n * s, cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemcpyAsync(ctx->pmat[0].p, mat, n * 4, cudaMemcpyDefault, st));
    if (n) k_iota<<<nblk(n, 256), 256, 0, st>>>(n, (int *)ctx->pid[0].p); ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(d2h_sync(ctx, st));
    return MPL_OK;
}

// Bring v / G into the order of x / F after a resample whose G2P has not run (mpl_ctx_s::vg_unsorted).
template <class T>
mpl_status sync_vg_order(mpl_ctx ctx) {
    if (!ctx->vg_unsorted) return MPL_OK;
    const int64_t np = ctx->np;
    const size_t s = sizeof(T);
    cudaStream_t st = ctx->stream;
    MPL_CHECK(ensure(ctx, ctx->pv_alt, np * 3 * s + 16));
    MPL_CHECK(ensure(ctx, ctx->pG_alt, np * 9 * s + 16));
    if (np) {
        k_vg_to_sorted<T><<<nblk(np, 256), 256, 0, st>>>(np, (const int *)ctx->pkey.p, (const int *)ctx->prank.p,
                                                        (const int *)ctx->t_bstart.p, (const T *)ctx->pv.p,
                                                        (const T *)ctx->pG.p, (T *)ctx->pv_alt.p, (T *)ctx->pG_alt.p);
        ctx->launches++;
        MPL_CUDA(cudaGetLastError());
    }
    std::swap(ctx->pv, ctx->pv_alt);
    std::swap(ctx->pG, ctx->pG_alt);
    ctx->vg_unsorted = false;
    return MPL_OK;
}
template mpl_status sync_vg_order<float>(mpl_ctx);
template mpl_status sync_vg_order<double>(mpl_ctx);

// ---- pipelined particle input (mpl_stage_particles) ------------------------------------------------
mpl_status io_streams(mpl_ctx ctx) {
    if (ctx->cstream) return MPL_OK;
    MPL_CUDA(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
    MPL_CUDA(cudaStreamCreateWithFlags(&ctx->rstream, cudaStreamNonBlocking));
    for (cudaEvent_t *e : {&ctx->ev_staged, &ctx->ev_adopted, &ctx->ev_rb_ready, &ctx->ev_rb_done})
        MPL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return MPL_OK;
}

// H2D of the next step's inputs into the staging set on the copy stream; it may only overwrite the
// staging buffers once the compute stream has adopted the previous staged set (ev_adopted), i.e. once
// the buffers swapped out then (the previous step's particle state) are no longer read.
template <class T>
mpl_status stage_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F, const void *G,
                           const void *vol, const int32_t *mat) {
    MPL_CHECK(io_streams(ctx));
    const size_t s = sizeof(T);
    if (ctx->staged) return MPL_ERR_STATE;  // one staged set at a time
    if (ctx->adopted_once) MPL_CUDA(cudaStreamWaitEvent(ctx->cstream, ctx->ev_adopted, 0));
    // the live set is resized on adoption; staging sizes follow n (both sets swap roles every step)
    MPL_CUDA(cudaStreamSynchronize(ctx->cstream));  // ensure() may free: nothing of ours in flight there
    MPL_CHECK(ensure(ctx, ctx->sx, n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->sv, n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->sF, n * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->sG, n * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->svol, n * s));
    MPL_CHECK(ensure(ctx, ctx->smat, n * 4));
    cudaStream_t cs = ctx->cstream;
    if (n) {
        MPL_CUDA(cudaMemcpyAsync(ctx->sx.p, x, n * 3 * s, cudaMemcpyDefault, cs));
        MPL_CUDA(cudaMemcpyAsync(ctx->sv.p, v, n * 3 * s, cudaMemcpyDefault, cs));
        MPL_CUDA(cudaMemcpyAsync(ctx->sF.p, F, n * 9 * s, cudaMemcpyDefault, cs));
        MPL_CUDA(cudaMemcpyAsync(ctx->sG.p, G, n * 9 * s, cudaMemcpyDefault, cs));
        MPL_CUDA(cudaMemcpyAsync(ctx->svol.p, vol, n * s, cudaMemcpyDefault, cs));
        MPL_CUDA(cudaMemcpyAsync(ctx->smat.p, mat, n * 4, cudaMemcpyDefault, cs));
    }
    MPL_CUDA(cudaEventRecord(ctx->ev_staged, cs));
    ctx->staged = true;
    ctx->staged_n = n;
    return MPL_OK;
}

// Called by mpl_resample: the compute stream waits for the staged copy, the staged set becomes the
// live particle set (buffer swap, no copy), the old live set becomes the staging set.
template <class T>
mpl_status adopt_staged(mpl_ctx ctx) {
    if (!ctx->staged) return MPL_OK;
    cudaStream_t st = ctx->stream;
    MPL_CUDA(cudaStreamWaitEvent(st, ctx->ev_staged, 0));
    const int64_t n = ctx->staged_n;
    const size_t s = sizeof(T);
    const int c = ctx->cur;
    // live buffers may be larger than n (ensure only grows): sizes of the swapped pairs are exchanged
    std::swap(ctx->px[c], ctx->sx);
    std::swap(ctx->pv, ctx->sv);
    std::swap(ctx->pF[c], ctx->sF);
    std::swap(ctx->pG, ctx->sG);
    std::swap(ctx->pvol[c], ctx->svol);
    std::swap(ctx->pmat[c], ctx->smat);
    ctx->np = n;
    ctx->np_own = n;
    ctx->vg_unsorted = false;  // the adopted set is in input order throughout
    const int nx = 1 - c;
    MPL_CHECK(ensure(ctx, ctx->px[nx], n * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->pF[nx], n * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->pvol[nx], n * s));
    MPL_CHECK(ensure(ctx, ctx->pmat[nx], n * 4));
    for (int i = 0; i < 2; i++) MPL_CHECK(ensure(ctx, ctx->pid[i], n * 4));
    MPL_CHECK(ensure(ctx, ctx->pkey, n * 4));
    MPL_CHECK(ensure(ctx, ctx->prank, n * 4));
    MPL_CHECK(ensure(ctx, ctx->pbase, n * 4));
    MPL_CHECK(ensure(ctx, ctx->prec, n * REC * s));
    if (n) k_iota<<<nblk(n, 256), 256, 0, st>>>(n, (int *)ctx->pid[c].p);
    ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    MPL_CUDA(cudaEventRecord(ctx->ev_adopted, st));
    ctx->adopted_once = true;
    ctx->staged = false;
    ctx->have_particles = true;
    return MPL_OK;
}

template mpl_status stage_particles<float>(mpl_ctx, int64_t, const void *, const void *, const void *, const void *,
                                           const void *, const int32_t *);
template mpl_status stage_particles<double>(mpl_ctx, int64_t, const void *, const void *, const void *, const void *,
                                            const void *, const int32_t *);
template mpl_status adopt_staged<float>(mpl_ctx);
template mpl_status adopt_staged<double>(mpl_ctx);

template <class T>
mpl_status resample_impl(mpl_ctx ctx, double dt) {
    cudaStream_t st = ctx->stream;
    const GridP &g = ctx->grid;
    const int N = g.nb[0] * g.nb[1] * g.nb[2];
    ctx->dense_n = N;
    ctx->dt = dt;
    MPL_CHECK(sync_vg_order<T>(ctx));  // a resample after a resample (no G2P in between)
    MPL_CHECK(redistribute_particles<T>(ctx));  // slab ranks: migration + ghosts (no-op on one rank)
    DBG_GUARDS("after redistribute");
    const int64_t np = ctx->np;
    int c = ctx->cur, nx = 1 - c;
#ifdef MPL_DEBUG
    // debug build: host-side consistency checks of the particle bookkeeping
    auto count_neg = [&](const void *pid, int64_t n, int64_t *neg) -> mpl_status {
        MPL_CHECK(d2h_sync(ctx, st));
        std::vector<int> h(n);
        if (n) MPL_CUDA(cudaMemcpy(h.data(), pid, n * 4, cudaMemcpyDeviceToHost));
        *neg = 0;
        for (int64_t i = 0; i < n; i++) *neg += h[i] < 0;
        return MPL_OK;
    };
    int64_t neg0 = 0;
    MPL_CHECK(count_neg(ctx->pid[c].p, np, &neg0));
    if (neg0 != np - ctx->np_own) {
        ctx->err = "debug: after redistribute " + std::to_string(neg0) + " ghosts, expected " +
                   std::to_string(np - ctx->np_own);
        fprintf(stderr, "[rank %d] %s\n", ctx->rank, ctx->err.c_str());
        return MPL_ERR_STATE;
    }
#endif
    {
        // per-particle scratch and the sorted-output buffer set (content not needed)
        const size_t sz = sizeof(T);
        MPL_CHECK(ensure(ctx, ctx->pkey, np * 4 + 16));
        MPL_CHECK(ensure(ctx, ctx->prank, np * 4 + 16));
        MPL_CHECK(ensure(ctx, ctx->pbase, np * 4 + 16));
        MPL_CHECK(ensure(ctx, ctx->prec, np * REC * sz + 16));
        MPL_CHECK(ensure(ctx, ctx->px[nx], np * 3 * sz + 16));
        MPL_CHECK(ensure(ctx, ctx->pF[nx], np * 9 * sz + 16));
        MPL_CHECK(ensure(ctx, ctx->pvol[nx], np * sz + 16));
        MPL_CHECK(ensure(ctx, ctx->pmat[nx], np * 4 + 16));
        MPL_CHECK(ensure(ctx, ctx->pid[nx], np * 4 + 16));
    }
    const int xlo = multi(ctx) ? ctx->slab_lo : -(1 << 30), xhi = multi(ctx) ? ctx->slab_hi : (1 << 30);
    DevScalars *sc = (DevScalars *)ctx->scalars.p;
    // reset error slots
    {
        DevScalars h{};
        h.oob_particle = 0x7fffffff;
        h.inv_particle = 0x7fffffff;
        h.cg_done_iter = -1;
        MPL_CUDA(cudaMemcpyAsync(sc, &h, sizeof h, cudaMemcpyHostToDevice, st));
    }
    MPL_CHECK(ensure(ctx, ctx->cflag, (size_t)N * 4));
    MPL_CHECK(ensure(ctx, ctx->nflag, (size_t)N * 4));
    MPL_CHECK(ensure(ctx, ctx->tile_of, (size_t)(N + 1) * 4));
    MPL_CUDA(cudaMemsetAsync(ctx->cflag.p, 0, (size_t)N * 4, st));
    MPL_CUDA(cudaMemsetAsync(ctx->nflag.p, 0, (size_t)N * 4, st));
    unsigned long long *counters = (unsigned long long *)((char *)ctx->scalars.p + 2048);
    MPL_CUDA(cudaMemsetAsync(counters, 0, 64, st));

    // a0: base cells + active cell blocks
    if (np) k_bin_flags<T><<<nblk(np, 256), 256, 0, st>>>(g, np, (const T *)ctx->px[c].p, (const int *)ctx->pid[c].p,
                                                         (int *)ctx->pbase.p, (int *)ctx->cflag.p, sc); ctx->launches++;
    DBG_GUARDS("resample #1");
    k_node_flags<<<nblk(N, 256), 256, 0, st>>>(g, (const int *)ctx->cflag.p, (int *)ctx->nflag.p, counters + 0, xlo,
                                               xhi); ctx->launches++;
    DBG_GUARDS("resample #2");
    MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->nflag.p, (int *)ctx->tile_of.p, N + 0));
    // fetch error flags + tile count (one sync)
    DevScalars hs;
    int last_tile = 0, last_flag = 0;
    MPL_CHECK(d2h(ctx, &hs, sc, sizeof hs, st));
    MPL_CHECK(d2h(ctx, &last_tile, (int *)ctx->tile_of.p + (N - 1), 4, st));
    MPL_CHECK(d2h(ctx, &last_flag, (int *)ctx->nflag.p + (N - 1), 4, st));
    unsigned long long nblocks = 0;
    MPL_CHECK(d2h(ctx, &nblocks, counters + 0, 8, st));
    MPL_CHECK(d2h_sync(ctx, st));
    mpl_status bad = MPL_OK;
    if (hs.oob_particle != 0x7fffffff) {
        ctx->err = "particle " + std::to_string(hs.oob_particle) +
                   " is out of the domain: its base cell must satisfy 0 <= b <= N-2 on every axis";
        bad = MPL_ERR_OUT_OF_DOMAIN;
    }
    MPL_CHECK(agree(ctx, bad));
    const int T_ = last_tile + last_flag;
    ctx->T = T_;
    ctx->n_blocks_active = (int64_t)nblocks;
    // tiles
    MPL_CHECK(ensure(ctx, ctx->t_coord, (size_t)T_ * 12 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_nplus, (size_t)T_ * 32 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_nminus, (size_t)T_ * 32 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_hascells, (size_t)T_ * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_cmask, (size_t)T_ * 8 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_cstart, (size_t)(T_ + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_bcount, ((size_t)T_ * 64 + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_bstart, ((size_t)T_ * 64 + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_cellof, (size_t)T_ * 64 * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_perm, (size_t)T_ * 64 + 16));
    k_tiles<<<nblk(N, 256), 256, 0, st>>>(g, (const int *)ctx->nflag.p, (int *)ctx->tile_of.p, (int *)ctx->t_coord.p); ctx->launches++;
    DBG_GUARDS("resample #3");
    if (T_) k_tile_nbrs<<<nblk(T_, 128), 128, 0, st>>>(g, T_, (const int *)ctx->t_coord.p, (const int *)ctx->tile_of.p,
                                                     (const int *)ctx->cflag.p, (int *)ctx->t_nplus.p,
                                                     (int *)ctx->t_nminus.p, (int *)ctx->t_hascells.p, xlo,
                                                     xhi); ctx->launches++;
    DBG_GUARDS("resample #4");
    MPL_CHECK(build_interface_lists(ctx));
    DBG_GUARDS("interface lists");
#ifdef MPL_DEBUG
    MPL_CHECK(debug_check_tiles(ctx, "after tile build"));
#endif
    // particle buckets: key = tile*64 + local base cell; counting sort
    MPL_CUDA(cudaMemsetAsync(ctx->t_bcount.p, 0, ((size_t)T_ * 64 + 1) * 4, st));
    if (np) k_count<<<nblk(np, 256), 256, 0, st>>>(g, np, (const int *)ctx->pbase.p, (const int *)ctx->tile_of.p,
                                                  (int *)ctx->pkey.p, (int *)ctx->prank.p, (int *)ctx->t_bcount.p); ctx->launches++;
    DBG_GUARDS("resample #5");
    MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->t_bcount.p, (int *)ctx->t_bstart.p, (int64_t)T_ * 64 + 1));
    // scatter into sorted order + records
    MPL_CHECK(ensure(ctx, ctx->pskey, (size_t)np * 4 + 16));
    if (np && sort_gather()) {
        MPL_CHECK(ensure(ctx, ctx->psrc, (size_t)np * 4 + 16));
        k_sort_src<<<nblk(np, 256), 256, 0, st>>>(np, (const int *)ctx->pkey.p, (const int *)ctx->prank.p,
                                                  (const int *)ctx->t_bstart.p, (int *)ctx->psrc.p);
        ctx->launches++;
        k_scatter_g<T><<<nblk(np, 256), 256, 0, st>>>(
            g, ctx->mats, np, (const int *)ctx->psrc.p, (const int *)ctx->pkey.p, (const T *)ctx->px[c].p,
            (const T *)ctx->pv.p, (const T *)ctx->pF[c].p, (const T *)ctx->pG.p, (const T *)ctx->pvol[c].p,
            (const int *)ctx->pmat[c].p, (const int *)ctx->pid[c].p, (T *)ctx->px[nx].p, (T *)ctx->pF[nx].p,
            (T *)ctx->pvol[nx].p, (int *)ctx->pmat[nx].p, (int *)ctx->pid[nx].p, (int *)ctx->pskey.p,
            (T *)ctx->prec.p, sc);
        ctx->launches++;
    } else if (np)
        k_scatter<T><<<nblk(np, 256), 256, 0, st>>>(
            g, ctx->mats, np, (const int *)ctx->pkey.p, (const int *)ctx->prank.p, (const int *)ctx->t_bstart.p,
            (const T *)ctx->px[c].p, (const T *)ctx->pv.p, (const T *)ctx->pF[c].p, (const T *)ctx->pG.p,
            (const T *)ctx->pvol[c].p, (const int *)ctx->pmat[c].p, (const int *)ctx->pid[c].p, (T *)ctx->px[nx].p,
            (T *)ctx->pF[nx].p, (T *)ctx->pvol[nx].p, (int *)ctx->pmat[nx].p, (int *)ctx->pid[nx].p,
            (int *)ctx->pskey.p, (T *)ctx->prec.p, sc); ctx->launches++;
    DBG_GUARDS("resample #6");
    ctx->cur = nx;
    ctx->vg_unsorted = np > 0;  // v / G follow order c until G2P (or sync_vg_order) rewrites them
#ifdef MPL_DEBUG
    {
        int bsum = 0;
        MPL_CHECK(d2h_sync(ctx, st));
        MPL_CHECK(d2h(ctx, &bsum, (int *)ctx->t_bstart.p + (size_t)T_ * 64, 4, st)); MPL_CHECK(d2h_sync(ctx, st));
        int64_t neg1 = 0;
        MPL_CHECK(count_neg(ctx->pid[nx].p, np, &neg1));
        if (bsum != np || neg1 != neg0) {
            ctx->err = "debug: bucket total " + std::to_string(bsum) + " (np " + std::to_string(np) + "), ghosts " +
                       std::to_string(neg1) + " after sort vs " + std::to_string(neg0) + ", T " + std::to_string(T_);
            fprintf(stderr, "[rank %d] %s\n", ctx->rank, ctx->err.c_str());
            return MPL_ERR_STATE;
        }
    }
#endif
    // structural cells: masks, padded counts, compact offsets
    MPL_CHECK(ensure(ctx, ctx->t_ccount, (size_t)(T_ + 1) * 4 + 16));
    MPL_CUDA(cudaMemsetAsync(ctx->t_ccount.p, 0, (size_t)(T_ + 1) * 4, st));
    MPL_CHECK(ensure(ctx, ctx->t_ncell, (size_t)(T_ + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_kcnt, (size_t)(T_ + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_kstart, (size_t)(T_ + 1) * 4 + 16));
    MPL_CUDA(cudaMemsetAsync(ctx->t_kcnt.p, 0, (size_t)(T_ + 1) * 4, st));
    MPL_CHECK(ensure(ctx, ctx->t_kcnt2, (size_t)(T_ + 1) * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_kstart2, (size_t)(T_ + 1) * 4 + 16));
    MPL_CUDA(cudaMemsetAsync(ctx->t_kcnt2.p, 0, (size_t)(T_ + 1) * 4, st));
    if (T_) k_cell_mask<<<T_, 64, 0, st>>>(g, T_, (const int *)ctx->t_coord.p, (const int *)ctx->t_nminus.p,
                                          (const int *)ctx->t_bcount.p, (const int *)ctx->t_hascells.p,
                                          (unsigned long long *)ctx->t_cmask.p,
                                          (int *)ctx->t_ccount.p, (int *)ctx->t_ncell.p, (int *)ctx->t_kcnt.p,
                                          counters + 1, (int *)ctx->t_kcnt2.p); ctx->launches++;
    DBG_GUARDS("resample #7");
    MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->t_ccount.p, (int *)ctx->t_cstart.p, (int64_t)T_ + 1));
    MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->t_kcnt.p, (int *)ctx->t_kstart.p, (int64_t)T_ + 1));
    MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->t_kcnt2.p, (int *)ctx->t_kstart2.p, (int64_t)T_ + 1));
    int Cpad = 0, Ktot = 0, Ktot2 = 0;
    MPL_CHECK(d2h(ctx, &Ktot, (int *)ctx->t_kstart.p + T_, 4, st));
    MPL_CHECK(d2h(ctx, &Ktot2, (int *)ctx->t_kstart2.p + T_, 4, st));
    unsigned long long ncells = 0;
    MPL_CHECK(d2h(ctx, &Cpad, (int *)ctx->t_cstart.p + T_, 4, st));
    MPL_CHECK(d2h(ctx, &ncells, counters + 1, 8, st));
    MPL_CHECK(d2h(ctx, &hs, sc, sizeof hs, st));
    MPL_CHECK(d2h_sync(ctx, st));
    bad = MPL_OK;
    if (hs.inv_particle != 0x7fffffff) {
        ctx->err = "particle " + std::to_string(hs.inv_particle) + " has det F_p <= 0 (inverted element)";
        bad = MPL_ERR_INVERTED;
    }
    if (agree(ctx, bad) != MPL_OK) {
        ctx->cur = c;  // particle state unchanged
        ctx->vg_unsorted = false;
        return bad != MPL_OK ? bad : MPL_ERR_STATE;
    }
    ctx->C = Cpad;
    ctx->n_cells_active = (int64_t)ncells;
    const int nm = ctx->mats.nmat;
    const size_t C = (size_t)Cpad + 4;
    size_t s = sizeof(T);
    MPL_CHECK(ensure(ctx, ctx->c_local, C));
    MPL_CHECK(ensure(ctx, ctx->q_m, C * s));
    MPL_CHECK(ensure(ctx, ctx->q_mv, C * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->q_mG, C * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->q_slot, C * nm * 16 * s));
    if (ctx->mats.plastic) MPL_CHECK(ensure(ctx, ctx->q_Sp, C * nm * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->q_vc, C * 12 * s));  // (v_c, G_c) per cell, written by Load's n2c
    MPL_CHECK(ensure(ctx, ctx->K, (size_t)std::max(Ktot, Ktot2) * s + 256));  // either tangent layout
    if (T_) {
        k_cell_list<<<T_, 64, 0, st>>>(T_, (const unsigned long long *)ctx->t_cmask.p, (const int *)ctx->t_cstart.p,
                                       (uint8_t *)ctx->c_local.p, (int *)ctx->t_cellof.p, (uint8_t *)ctx->t_perm.p);
        ctx->launches++;
    DBG_GUARDS("resample #8");
        if (p2q_scatter()) {
            // zeroed accumulators, one CTA per tile scattering its particles, then the per-slot finish
            MPL_CUDA(cudaMemsetAsync(ctx->q_m.p, 0, C * s, st));
            MPL_CUDA(cudaMemsetAsync(ctx->q_mv.p, 0, C * 3 * s, st));
            MPL_CUDA(cudaMemsetAsync(ctx->q_mG.p, 0, C * 9 * s, st));
            MPL_CUDA(cudaMemsetAsync(ctx->q_slot.p, 0, C * nm * 16 * s, st));
#define P2QT_ARGS                                                                                           \
    g, ctx->mats, (const int *)ctx->t_coord.p, (const int *)ctx->t_nplus.p, (const int *)ctx->t_bstart.p, \
        (const int *)ctx->t_cellof.p, (const T *)ctx->prec.p, (T *)ctx->q_m.p, (T *)ctx->q_mv.p,           \
        (T *)ctx->q_mG.p, (T *)ctx->q_slot.p
            // dense buckets (MPL_P2Q_HI: 0 off, 1 on, default when np / cells >= P2Q_HI_PPC): k_p2q_hi
            static int hi_mode = -1;
            if (hi_mode < 0) {
                const char *e = getenv("MPL_P2Q_HI");
                hi_mode = e ? (e[0] == '1' ? 1 : 0) : 2;
            }
            const bool hi = nm <= 2 && (hi_mode == 1 || (hi_mode == 2 && ncells > 0 &&
                                                        (double)ctx->np >= P2Q_HI_PPC * (double)ncells));
            if (hi) {
                const size_t sm = (size_t)(13 + 7 * (nm == 1 ? 1 : 2)) * 8 * 68 * s + (size_t)8 * 2 * 32 * REC * s;
                if (nm == 1) {
                    MPL_CUDA(cudaFuncSetAttribute(k_p2q_hi<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                    k_p2q_hi<T, 1><<<T_, 256, sm, st>>>(P2QT_ARGS);
                } else {
                    MPL_CUDA(cudaFuncSetAttribute(k_p2q_hi<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                    k_p2q_hi<T, 2><<<T_, 256, sm, st>>>(P2QT_ARGS);
                }
            } else if (nm == 1) {
                const size_t sm = (((size_t)125 * P2QNV<1>::V + 3) & ~(size_t)3) * s + (size_t)2 * P2Q_CAP * REC * s;
                MPL_CUDA(cudaFuncSetAttribute(k_p2q_tile<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                k_p2q_tile<T, 1><<<T_, 256, sm, st>>>(P2QT_ARGS);
            } else if (nm <= 2) {
                const size_t sm = (((size_t)125 * P2QNV<2>::V + 3) & ~(size_t)3) * s + (size_t)2 * P2Q_CAP * REC * s;
                MPL_CUDA(cudaFuncSetAttribute(k_p2q_tile<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                k_p2q_tile<T, 2><<<T_, 256, sm, st>>>(P2QT_ARGS);
            } else {
                const size_t sm = (((size_t)125 * P2QNV<MPL_MAXMAT>::V + 3) & ~(size_t)3) * s + (size_t)2 * P2Q_CAP * REC * s;
                MPL_CUDA(cudaFuncSetAttribute(k_p2q_tile<T, MPL_MAXMAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sm));
                k_p2q_tile<T, MPL_MAXMAT><<<T_, 256, sm, st>>>(P2QT_ARGS);
            }
#undef P2QT_ARGS
            ctx->launches++;
            MPL_CUDA(cudaGetLastError());
            const int64_t NS = (int64_t)Cpad * nm;
            k_p2q_finish<T><<<nblk(NS, 128), 128, 0, st>>>((int64_t)Cpad, ctx->mats, (const uint8_t *)ctx->c_local.p,
                                                           (T *)ctx->q_slot.p,
                                                           ctx->mats.plastic ? (T *)ctx->q_Sp.p : (T *)nullptr, sc);
            ctx->launches++;
        } else {
#define P2Q_ARGS                                                                                             \
    g, ctx->mats, (const int *)ctx->t_coord.p, (const int *)ctx->t_nminus.p, (const int *)ctx->t_bstart.p, \
        (const int *)ctx->t_cellof.p, (const T *)ctx->prec.p, (T *)ctx->q_m.p, (T *)ctx->q_mv.p,            \
        (T *)ctx->q_mG.p, (T *)ctx->q_slot.p, ctx->mats.plastic ? (T *)ctx->q_Sp.p : (T *)nullptr, sc
        if (ctx->mats.nmat <= 2) k_p2q8<T, 2><<<2 * T_, 256, 0, st>>>(P2Q_ARGS);
        else k_p2q8<T, MPL_MAXMAT><<<2 * T_, 256, 0, st>>>(P2Q_ARGS);
#undef P2Q_ARGS
        ctx->launches++;
        }
    DBG_GUARDS("resample #9");
    }
    ctx->multi_slot_cells = 0;
    ctx->nonid_base_cells = 0;
    if (Cpad) {
        k_multislot<T><<<nblk(Cpad, 256), 256, 0, st>>>((int64_t)Cpad, nm, (const uint8_t *)ctx->c_local.p,
                                                       (const T *)ctx->q_slot.p, counters + 3, counters + 4);
        ctx->launches++;
    }
    // nodes
    const size_t NN = (size_t)T_ * 64 + 64;
    MPL_CHECK(ensure(ctx, ctx->n_mass, NN * s));
    MPL_CHECK(ensure(ctx, ctx->n_flag, NN));
    DevBuf *vecs[] = {&ctx->n_vn, &ctx->n_vhat, &ctx->n_v, &ctx->n_vt, &ctx->n_g, &ctx->n_diag,
                      &ctx->n_x, &ctx->n_r, &ctx->n_u, &ctx->n_u2};  // n_p (p + Hp): newton_impl
    for (DevBuf *b : vecs) MPL_CHECK(ensure(ctx, *b, NN * 4 * s));
    MPL_CHECK(ensure(ctx, ctx->n_act, NN * 4));
    MPL_CHECK(ensure(ctx, ctx->n_own, NN));
    if (multi(ctx)) MPL_CHECK(ensure(ctx, ctx->n_mown, NN * s));
    MPL_CHECK(ensure(ctx, ctx->n_canon, NN * 4));
    MPL_CHECK(ensure(ctx, ctx->n_list, NN * 4));
#define C2N_ARGS                                                                                                  \
    g, ctx->boxes, dt, ctx->gravity[0], ctx->gravity[1], ctx->gravity[2], (const int *)ctx->t_coord.p,            \
        (const int *)ctx->t_nminus.p, (const int *)ctx->t_cellof.p, (const int *)ctx->t_hascells.p,                \
        (const T *)ctx->q_m.p, (const T *)ctx->q_mv.p, (const T *)ctx->q_mG.p, (T *)ctx->n_mass.p,                \
        (uint8_t *)ctx->n_flag.p, (vec4<T> *)ctx->n_vn.p, (vec4<T> *)ctx->n_vhat.p, (vec4<T> *)ctx->n_v.p,          \
        (uint8_t *)ctx->n_own.p, (T *)ctx->n_mown.p, counters + 2
    if (!multi(ctx)) {
        if (T_) k_c2n<T, 0><<<T_, 64, 0, st>>>(C2N_ARGS), ctx->launches++;
    DBG_GUARDS("resample #10");
    } else {
        if (T_) k_c2n<T, 1><<<T_, 64, 0, st>>>(C2N_ARGS), ctx->launches++;
    DBG_GUARDS("resample #11");
        MPL_CHECK(c2n_halo<T>(ctx));
        DBG_GUARDS("c2n_halo");
        if (T_) k_c2n<T, 2><<<T_, 64, 0, st>>>(C2N_ARGS), ctx->launches++;
    DBG_GUARDS("resample #12");
    }
#undef C2N_ARGS
    const int64_t NT = (int64_t)T_ * 64;
    int nact = 0;
    if (NT) {
        k_node_active<<<nblk(NT, 256), 256, 0, st>>>(NT, (const uint8_t *)ctx->n_flag.p, (int *)ctx->n_act.p); ctx->launches++;
    DBG_GUARDS("resample #13");
        MPL_CHECK(exclusive_scan<int>(ctx, (const int *)ctx->n_act.p, (int *)ctx->n_canon.p, NT));
        int lc = 0, la = 0;  // read before k_node_canon rewrites inactive entries (stream order)
        MPL_CHECK(d2h(ctx, &lc, (int *)ctx->n_canon.p + (NT - 1), 4, st));
        MPL_CHECK(d2h(ctx, &la, (int *)ctx->n_act.p + (NT - 1), 4, st));
        k_node_canon<<<nblk(NT, 256), 256, 0, st>>>(NT, (const uint8_t *)ctx->n_flag.p, (int *)ctx->n_canon.p,
                                                    (int *)ctx->n_list.p); ctx->launches++;
    DBG_GUARDS("resample #14");
        MPL_CHECK(d2h_sync(ctx, st));
        nact = lc + la;
        unsigned long long nf = 0, ms = 0, ni = 0;
        MPL_CHECK(d2h(ctx, &nf, counters + 2, 8, st));
        MPL_CHECK(d2h(ctx, &ms, counters + 3, 8, st));
        MPL_CHECK(d2h(ctx, &ni, counters + 4, 8, st));
        MPL_CHECK(d2h_sync(ctx, st));
        ctx->n_free_nodes = (int64_t)nf;
        ctx->multi_slot_cells = (int64_t)ms;
        ctx->nonid_base_cells = (int64_t)ni;
    }
    ctx->n_nodes_active = nact;
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(d2h_sync(ctx, st));
    {
        int nf = 0;
        MPL_CHECK(d2h(ctx, &nf, &sc->nonfinite, sizeof nf, st)); MPL_CHECK(d2h_sync(ctx, st));
        mpl_status bad2 = MPL_OK;
        if (nf) {
            ctx->err = "a quadrature stress lies outside the split Neo-Hookean inversion domain "
                       "(1 + 2 tr(tau) / (3 kappa) <= 0 or no admissible stretch; P:268, App. C)";
            bad2 = MPL_ERR_INVERSION_DOMAIN;
        }
        MPL_CHECK(agree(ctx, bad2));
    }
#ifdef MPL_DEBUG
    MPL_CHECK(debug_check_tiles(ctx, "end of resample"));
#endif
    ctx->resampled = true;
    ctx->linearized = false;
    ctx->solved = false;
    return MPL_OK;
}

template mpl_status import_particles<float>(mpl_ctx, int64_t, const void *, const void *, const void *,
                                            const void *, const void *, const int32_t *);
template mpl_status import_particles<double>(mpl_ctx, int64_t, const void *, const void *, const void *,
                                             const void *, const void *, const int32_t *);
template mpl_status resample_impl<float>(mpl_ctx, double);
template mpl_status resample_impl<double>(mpl_ctx, double);
