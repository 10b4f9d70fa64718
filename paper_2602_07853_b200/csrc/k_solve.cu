#include <array>
// k_solve.cu — SURVEY §8(a) rows a5-a8: linearisation (energy / gradient / cached tangent /
// Jacobi diagonal), the matrix-free HVP, Jacobi-PCG vector kernels and the Newton driver.
//
// Paper: incremental potential Eq. incpot-rotfree, trial F_c(v) = (I + dt G_c(v)) S_c
// (Eq. Ftrial-rotfree, Eq. rotfree-def), StVK-Hencky energy (Eq. hencky-energy
// P:192-195), gradient / Hessian of App. B, G_c = sum_i v_i (x) grad w_ic
// with grad w_ic = (x_i - x_c)/(2 dx^2), "matrix-free PCG".
//
// Tile kernels: one CTA per 4^3 node block ("tile").  The CTA stages the 5^3 node halo of its cell
// block in shared memory, evaluates its (<= 64) quadrature points, then reduces the per-cell nodal
// contributions with a shared-memory gather per node.  Nodes whose 8 cells all lie in the tile
// (local coords 1..3) are written with plain stores; the other (face) nodes are summed with global
// atomics into a zeroed output.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include <type_traits>

#include "mpl_common.cuh"

namespace {

__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

// halo index h in 5^3 -> (tile, local) of the node; returns -1 if the neighbour tile is absent
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

// =============================================================================================
// Per-cell PSD projection of the tangent ("per-cell PSD projection of the elastic energy
// Hessian (eigenvalue clamping at 0)"; the paper's "off-the-shelf nonlinear solvers" P:4, "trust
// region ... damping/line-search" P:1150).  K (9x9 symmetric, packed upper triangle, 45 reals) is
// replaced by Q max(Lambda, 0) Q^T, with (Lambda, Q) from a cyclic Jacobi eigen-decomposition in fp64
// (a continuous map of K: no per-cell decision, and a positive-definite K is returned up to rounding).
// Used when the exact Hessian is indefinite (compressed StVK-Hencky cells: cfg5's plate contact).
// =============================================================================================
// Register-resident cyclic Jacobi on the packed upper triangle a[45] (A <- J^T A J, V <- V J per pair
// (p, q); Numerical Recipes' update form), every index compile-time so nothing spills to local memory;
// in the context's precision (fp32 resolves the eigenvalues to ~eps |K|, well inside the parity bars).
template <class T>
__device__ __forceinline__ void psd_project45(T *k) {
    T a[45], V[81];
#pragma unroll
    for (int e = 0; e < 45; e++) a[e] = k[e];
#pragma unroll
    for (int e = 0; e < 81; e++) V[e] = (e % 10 == 0) ? T(1) : T(0);
    T nd = T(0);
#pragma unroll
    for (int r = 0; r < 9; r++) nd += a[kidx(r, r)] * a[kidx(r, r)];
    const T tiny = (sizeof(T) == 4 ? T(1e-14) : T(1e-30)) * nd;
    for (int sweep = 0; sweep < 12; sweep++) {
        T off = T(0);
#pragma unroll
        for (int p_ = 0; p_ < 8; p_++)
#pragma unroll
            for (int q = p_ + 1; q < 9; q++) off += a[kidx(p_, q)] * a[kidx(p_, q)];
        if (!(off > tiny)) break;
#pragma unroll
        for (int p_ = 0; p_ < 8; p_++)
#pragma unroll
            for (int q = p_ + 1; q < 9; q++) {
                const T apq = a[kidx(p_, q)];
                if (apq != T(0)) {
                    const T th = (a[kidx(q, q)] - a[kidx(p_, p_)]) / (T(2) * apq);
                    const T t = (th >= T(0) ? T(1) : T(-1)) / (fabs(th) + sqrt(th * th + T(1)));
                    const T c = T(1) / sqrt(t * t + T(1)), s_ = t * c, tau = s_ / (T(1) + c);
                    a[kidx(p_, p_)] -= t * apq;
                    a[kidx(q, q)] += t * apq;
                    a[kidx(p_, q)] = T(0);
#pragma unroll
                    for (int r = 0; r < 9; r++) {
                        if (r == p_ || r == q) continue;
                        const int ip = r < p_ ? kidx(r, p_) : kidx(p_, r), iq = r < q ? kidx(r, q) : kidx(q, r);
                        const T arp = a[ip], arq = a[iq];
                        a[ip] = arp - s_ * (arq + tau * arp);
                        a[iq] = arq + s_ * (arp - tau * arq);
                    }
#pragma unroll
                    for (int r = 0; r < 9; r++) {
                        const T vrp = V[9 * r + p_], vrq = V[9 * r + q];
                        V[9 * r + p_] = vrp - s_ * (vrq + tau * vrp);
                        V[9 * r + q] = vrq + s_ * (vrp - tau * vrq);
                    }
                }
            }
    }
    T lam[9];
#pragma unroll
    for (int i = 0; i < 9; i++) lam[i] = a[kidx(i, i)] > T(0) ? a[kidx(i, i)] : T(0);
#pragma unroll
    for (int r = 0; r < 9; r++)
#pragma unroll
        for (int c = r; c < 9; c++) {
            T v = T(0);
#pragma unroll
            for (int i = 0; i < 9; i++) v += V[9 * r + i] * lam[i] * V[9 * c + i];
            k[kidx(r, c)] = v;
        }
}

// unit quaternion (w, x, y, z) of a proper rotation matrix R (row-major), Shepperd's branch choice
template <class T>
__device__ __forceinline__ void rot_quat(const T R[9], T q[4]) {
    const T tr = R[0] + R[4] + R[8];
    T w, x, y, z;
    if (tr > T(0)) {
        const T s = T(2) * sqrt(tr + T(1));
        w = T(0.25) * s; x = (R[7] - R[5]) / s; y = (R[2] - R[6]) / s; z = (R[3] - R[1]) / s;
    } else if (R[0] > R[4] && R[0] > R[8]) {
        const T s = T(2) * sqrt(T(1) + R[0] - R[4] - R[8]);
        w = (R[7] - R[5]) / s; x = T(0.25) * s; y = (R[1] + R[3]) / s; z = (R[2] + R[6]) / s;
    } else if (R[4] > R[8]) {
        const T s = T(2) * sqrt(T(1) + R[4] - R[0] - R[8]);
        w = (R[2] - R[6]) / s; x = (R[1] + R[3]) / s; y = T(0.25) * s; z = (R[5] + R[7]) / s;
    } else {
        const T s = T(2) * sqrt(T(1) + R[8] - R[0] - R[4]);
        w = (R[3] - R[1]) / s; x = (R[2] + R[6]) / s; y = (R[5] + R[7]) / s; z = T(0.25) * s;
    }
    const T n = rsqrt(w * w + x * x + y * y + z * z);
    q[0] = w * n; q[1] = x * n; q[2] = y * n; q[3] = z * n;
}

// =============================================================================================
// a5 / a8: linearisation.  MODE = LIN_ENERGY (Phi only), LIN_GRAD (+ g), LIN_FULL (+ K, diag).
// =============================================================================================
// HONLY: every material slot is elastic StVK-Hencky (the other laws and the plastic base update are
// compiled out: a third of the code, and ncu showed 20 % instruction-fetch stalls on the general kernel)
// LMINB > 1: 64-thread launch with LMINB CTAs per SM requested from ptxas (the Hencky-only full
// linearisation at 12: 80 registers, small spills, 24 warps / SM: cfg4 3.89 -> 3.62 ms per step; 16: 3.84)
template <class T, int MODE, bool HONLY = false, int LMINB = 1, bool PSD = false, bool KCT = false>
__global__ void __launch_bounds__(LMINB > 1 ? 64 : 128, LMINB) k_linearize(GridP g, MatP mp, double dt_, const int *__restrict__ nplus,
                                                   const int *__restrict__ cstart, const uint8_t *__restrict__ clocal,
                                                   const int *__restrict__ hascells, const vec4<T> *__restrict__ v,
                                                   const vec4<T> *__restrict__ vhat, const T *__restrict__ nmass,
                                                   const T *__restrict__ qslot, T *__restrict__ Kout,
                                                   const int *__restrict__ kstart, const int *__restrict__ ncell,
                                                   vec4<T> *__restrict__ grad, vec4<T> *__restrict__ diag,
                                                   T *__restrict__ qsp, DevScalars *sc, int kz, int kc) {
    constexpr int KS = (MODE == LIN_FULL) ? 64 * 45 : 1;
    // compressed tangent (kc = 1: fp32, every slot elastic StVK-Hencky, one occupied slot per cell):
    // KC_REALS (24) reals per cell, written in k_hvp_wz's interleaved pair layout
    // with PSD only when every base S is I (the resample counts the other cells): then K = c C(A) exactly, and
    // its per-cell projection is the blockwise clamping of C in the SVD frame
    // (a template instance per format: each carries only its own tangent code, see DESIGN §5 linearize)
    constexpr bool KC = KCT && (MODE == LIN_FULL) && HONLY && sizeof(T) == 4;
    DASSERT(kc == (KC ? 1 : 0));
    __shared__ unsigned int pm_s, cm_s[2];  // KC: k_hvp_wz lanes holding a cell; the tile's cell mask
    __shared__ vec4<T> vh[125];
    __shared__ T Pg[64 * 9];
    __shared__ T Ks[KS];
    __shared__ int cslot[64];
    __shared__ int zslot[MODE == LIN_FULL ? 64 : 1];
    const int t = blockIdx.x, tid = threadIdx.x;
    const int has = hascells[t];
    const int cs = cstart[t], nc = cstart[t + 1] - cs;
    DASSERT(nc >= 0 && nc <= 64 && cstart[t + 1] <= cstart[gridDim.x]);
    for (int h = tid; h < 125; h += blockDim.x) {
        int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        bool owned = hx < 4 && hy < 4 && hz < 4;
        int64_t n = (has || owned) ? halo_node(t, nplus, h) : -1;
        DASSERT(n < (int64_t)gridDim.x * 64);
        vh[h] = n >= 0 ? v[n] : mk4<T>(0, 0, 0, 0);
    }
    if (tid < 64) cslot[tid] = -1;
    if (MODE == LIN_FULL)
        for (int i = tid; i < nc * 45; i += blockDim.x) Ks[i] = T(0);
    if (tid == 0) { pm_s = 0u; cm_s[0] = cm_s[1] = 0u; }
    __syncthreads();
    if (has && tid < nc) {
        int l = clocal[cs + tid];
        if (l != 0xFF) {
            cslot[l] = tid;
            if (KC) {
                atomicOr(&pm_s, 1u << (kz_key(l) & 31));
                atomicOr(&cm_s[l >> 5], 1u << (l & 31));
            }
        }
    }
    if (KC) __syncthreads();  // pair slots known before the cell phase writes the compressed tangent
    // KC: element e of this cell at Kout[kc_base + (e / 2) * 4 np + 2 (e & 1)] (pair layout)
    int64_t kc_base = 0;
    int kc_np = 0;
    if (KC && has && tid < nc && clocal[cs + tid] != 0xFF) {
        const int l = clocal[cs + tid], lane = kz_key(l) & 31;
        kc_np = __popc(pm_s);
        kc_base = kstart[t] + (int64_t)__popc(pm_s & ((1u << lane) - 1u)) * 4 + (l & 1);
        DASSERT(kstart[t] + 2 * KC_REALS * kc_np <= kstart[t + 1]);
        // the lane's other cell (l ^ 1: the other z of the pair) absent: its half of the pair slot is zero
        if (!((cm_s[(l ^ 1) >> 5] >> ((l ^ 1) & 31)) & 1u))
            for (int e = 0; e < KC_REALS; e++) Kout[kc_base + (int64_t)(e >> 1) * 4 * kc_np + 2 * (e & 1) + (1 - 2 * (l & 1))] = T(0);
    }
    bool kc_done = false;
    double e_loc = 0.0;
    const T dt = T(dt_);
    const T q = T(0.25 * g.inv_dx);  // grad w = s q, s in {-1,+1}^3
    if (has && tid < nc) {
        int l = clocal[cs + tid];
        if (l != 0xFF) {
            int lx = l >> 4, ly = (l >> 2) & 3, lz = l & 3;
            T Gs[9];
#pragma unroll
            for (int a = 0; a < 9; a++) Gs[a] = T(0);
#pragma unroll
            for (int o = 0; o < 8; o++) {
                int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                vec4<T> u = vh[((lx + ox) * 5 + ly + oy) * 5 + lz + oz];
                T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
                Gs[0] += u.x * s0; Gs[1] += u.x * s1; Gs[2] += u.x * s2;
                Gs[3] += u.y * s0; Gs[4] += u.y * s1; Gs[5] += u.y * s2;
                Gs[6] += u.z * s0; Gs[7] += u.z * s1; Gs[8] += u.z * s2;
            }
            T W[9], A[9], AiT[9];  // W = dt G, A = I + W
#pragma unroll
            for (int a = 0; a < 9; a++) { W[a] = dt * q * Gs[a]; A[a] = W[a] + ((a % 4 == 0) ? T(1) : T(0)); }
            T detA = inv_transpose3(A, AiT);
            if (!(detA > T(0))) sc->inv_any = 1.0;  // amb-21: Phi = +inf
            T Pc[9];
#pragma unroll
            for (int a = 0; a < 9; a++) Pc[a] = T(0);
            const int nmat = mp.nmat;
            const int j = tid;
            for (int k = 0; k < nmat; k++) {
                const T *sl = qslot + ((int64_t)(cs + tid) * nmat + k) * 16;
                T V = sl[0];
                if (V == T(0)) continue;
                T mu = T(mp.mu[k]), lamL = T(mp.lam[k]);
                T E[9] = {sl[1], sl[4], sl[6], sl[4], sl[2], sl[5], sl[6], sl[5], sl[3]};
                if (!HONLY && qsp && mp.sigy[k] > 0.0) {
                    // fixed-point plasticity: the slot's base for this Newton iteration.
                    // Energy-only evaluations (line search) use the stored iterate base; the gradient /
                    // full linearisation at a new iterate v re-project: F^tr = A(v) S_base, F^E = F^tr P,
                    // S = S_base P  ->  E = S - I = (P - I) + E_base + E_base (P - I).
                    T *sp = qsp + ((int64_t)(cs + tid) * nmat + k) * 9;
                    if (MODE == LIN_ENERGY) {
#pragma unroll
                        for (int a = 0; a < 9; a++) E[a] = sp[a];
                    } else {
                        T WE0[9], Ht[9], Pm1[9], EP[9];
                        mm3(W, E, WE0);
#pragma unroll
                        for (int a = 0; a < 9; a++) Ht[a] = W[a] + E[a] + WE0[a];  // F^tr - I
                        vm_plastic_Pm1(Ht, mu, T(mp.sigy[k]), Pm1);
                        mm3(E, Pm1, EP);
#pragma unroll
                        for (int a = 0; a < 9; a++) {
                            E[a] = Pm1[a] + E[a] + EP[a];
                            sp[a] = E[a];
                        }
                    }
                }
                // H = F - I = W + E + W E
                T WE[9], H[9];
                mm3(W, E, WE);
#pragma unroll
                for (int a = 0; a < 9; a++) H[a] = W[a] + E[a] + WE[a];
                // b - I = H + H^T + H H^T
                T B[9];
#pragma unroll
                for (int a = 0; a < 3; a++)
#pragma unroll
                    for (int b = a; b < 3; b++) {
                        T val = H[3 * a + b] + H[3 * b + a] + H[3 * a] * H[3 * b] + H[3 * a + 1] * H[3 * b + 1] +
                                H[3 * a + 2] * H[3 * b + 2];
                        B[3 * a + b] = val;
                        B[3 * b + a] = val;
                    }
                if (!HONLY && mp.kind[k] == 2) {
                    // ---- J-based water slot (PAPER §4.5): psi = kappa/2 (J-1)^2, J = det(A S),
                    //      tau = pi I, pi = kappa J (J-1); column (a,b): dJ/J = dt (F^{-T} S)[a][b],
                    //      dtau = kappa (2J-1) J (dJ/J) I ----
                    const T kap = T(mp.kappa[k]);
                    const T jm1 = det_ipm1(H), Jv = T(1) + jm1;
                    e_loc += (double)(V * T(0.5) * kap * jm1 * jm1);
                    if (MODE == LIN_ENERGY) continue;
                    const T pi = kap * Jv * jm1;
                    T TA[9];  // tau A^{-T}
#pragma unroll
                    for (int a = 0; a < 9; a++) TA[a] = pi * AiT[a];
                    const T sV = dt * V;
#pragma unroll
                    for (int a = 0; a < 9; a++) Pc[a] += sV * TA[a];
                    if (MODE == LIN_FULL) {
                        T F[9], S[9], FiT[9], M[9];
#pragma unroll
                        for (int a = 0; a < 9; a++) {
                            F[a] = H[a] + ((a % 4 == 0) ? T(1) : T(0));
                            S[a] = E[a] + ((a % 4 == 0) ? T(1) : T(0));
                        }
                        inv_transpose3(F, FiT);
                        mm3(FiT, S, M);
                        const T kscale = sV * T(1.0 / 16.0) * T(g.inv_dx * g.inv_dx);
                        const T dpi_c = kap * (T(2) * Jv - T(1)) * Jv * dt;
                        T *Kr = Ks + j * 45;
#pragma unroll
                        for (int a = 0; a < 3; a++)
#pragma unroll
                            for (int b = 0; b < 3; b++) {
                                const T dpi = dpi_c * M[3 * a + b];
                                const int cidx = 3 * a + b;
#pragma unroll
                                for (int i = 0; i < 3; i++)
#pragma unroll
                                    for (int jj = 0; jj < 3; jj++) {
                                        T r1 = dpi * AiT[3 * i + jj];
                                        T r2 = -dt * TA[3 * i + b] * AiT[3 * a + jj];
                                        T val = kscale * (r1 + r2);
                                        const int r = 3 * i + jj;
                                        if (r == cidx) Kr[kidx(r, r)] += val;
                                        else if (r < cidx) Kr[kidx(r, cidx)] += T(0.5) * val;
                                        else Kr[kidx(cidx, r)] += T(0.5) * val;
                                    }
                            }
                    }
                    continue;
                }
                if (!HONLY && mp.kind[k] == 1) {
                    // ---- split Neo-Hookean slot (PAPER §4.3.2; stable forms in mpl_common.cuh) ----
                    const T kap = T(mp.kappa[k]);
                    const T jm1 = det_ipm1(H), j23 = mexpm1(T(-2.0 / 3.0) * mlog1p(jm1));
                    const T trB = B[0] + B[4] + B[8];
                    const T psi = T(0.5) * mu * (T(3) * j23 + trB * (T(1) + j23)) + T(0.25) * kap * nh_f(jm1);
                    e_loc += (double)(V * psi);
                    if (MODE == LIN_ENERGY) continue;
                    const T sdev = mu * (T(1) + j23), al = T(0.5) * kap * jm1 * (T(2) + jm1);
                    T devB[9], tau[9];
#pragma unroll
                    for (int a = 0; a < 9; a++) {
                        devB[a] = B[a] - ((a % 4 == 0) ? trB / T(3) : T(0));
                        tau[a] = sdev * devB[a] + ((a % 4 == 0) ? al : T(0));
                    }
                    T TA[9];  // tau A^{-T}
                    mm3(tau, AiT, TA);
                    const T sV = dt * V;
#pragma unroll
                    for (int a = 0; a < 9; a++) Pc[a] += sV * TA[a];
                    if (MODE == LIN_FULL) {
                        // column (a,b) of the tangent: dF = dt e_a (x) S[b,:] (dG = e_a e_b^T), so
                        //   dJ = J dt (F^{-T} S)[a][b], db = dt (e_a y_b^T + y_b e_a^T), y_b = (F S)[:, b],
                        //   dtau = mu J^{-2/3} (-2/3 dJ/J dev(b) + dev(db)) + kappa J dJ I.
                        T F[9], S[9], FS[9], FiT[9], M[9];
#pragma unroll
                        for (int a = 0; a < 9; a++) {
                            F[a] = H[a] + ((a % 4 == 0) ? T(1) : T(0));
                            S[a] = E[a] + ((a % 4 == 0) ? T(1) : T(0));
                        }
                        mm3(F, S, FS);
                        inv_transpose3(F, FiT);
                        mm3(FiT, S, M);
                        const T Jv = T(1) + jm1;
                        const T kscale = sV * T(1.0 / 16.0) * T(g.inv_dx * g.inv_dx);
                        T *Kr = Ks + j * 45;
#pragma unroll
                        for (int a = 0; a < 3; a++)
#pragma unroll
                            for (int b = 0; b < 3; b++) {
                                const T dJ_J = dt * M[3 * a + b];  // dJ / J
                                const T tdb3 = T(2.0 / 3.0) * dt * FS[3 * a + b];
                                T dtau[9];
#pragma unroll
                                for (int i = 0; i < 3; i++)
#pragma unroll
                                    for (int jj = 0; jj < 3; jj++) {
                                        T db = dt * ((i == a ? FS[3 * jj + b] : T(0)) + (jj == a ? FS[3 * i + b] : T(0)));
                                        if (i == jj) db -= tdb3;  // dev(db)
                                        dtau[3 * i + jj] = sdev * (T(-2.0 / 3.0) * dJ_J * devB[3 * i + jj] + db) +
                                                           ((i == jj) ? kap * Jv * Jv * dJ_J : T(0));
                                    }
                                const int cidx = 3 * a + b;
#pragma unroll
                                for (int i = 0; i < 3; i++)
#pragma unroll
                                    for (int jj = 0; jj < 3; jj++) {
                                        T r1 = dtau[3 * i] * AiT[jj] + dtau[3 * i + 1] * AiT[3 + jj] + dtau[3 * i + 2] * AiT[6 + jj];
                                        T r2 = -dt * TA[3 * i + b] * AiT[3 * a + jj];
                                        T val = kscale * (r1 + r2);
                                        const int r = 3 * i + jj;
                                        if (r == cidx) Kr[kidx(r, r)] += val;
                                        else if (r < cidx) Kr[kidx(r, cidx)] += T(0.5) * val;
                                        else Kr[kidx(cidx, r)] += T(0.5) * val;
                                    }
                            }
                    }
                    continue;
                }
                T lam3[3], Q[9];
                sym_eig3(B, lam3, Q);
                T l0 = mlog1p(lam3[0]), l1 = mlog1p(lam3[1]), l2 = mlog1p(lam3[2]);
                T sl_ = l0 + l1 + l2;
                T psi = T(0.25) * mu * (l0 * l0 + l1 * l1 + l2 * l2) + T(0.125) * lamL * sl_ * sl_;
                e_loc += (double)(V * psi);
                if (MODE == LIN_ENERGY) continue;
                T tp[3] = {mu * l0 + T(0.5) * lamL * sl_, mu * l1 + T(0.5) * lamL * sl_, mu * l2 + T(0.5) * lamL * sl_};
                T tau[9];
#pragma unroll
                for (int a = 0; a < 3; a++)
#pragma unroll
                    for (int b = 0; b < 3; b++)
                        tau[3 * a + b] = Q[3 * a] * Q[3 * b] * tp[0] + Q[3 * a + 1] * Q[3 * b + 1] * tp[1] +
                                         Q[3 * a + 2] * Q[3 * b + 2] * tp[2];
                T TA[9];  // tau A^{-T}
                mm3(tau, AiT, TA);
                const T sV = dt * V;
#pragma unroll
                for (int a = 0; a < 9; a++) Pc[a] += sV * TA[a];
                if (MODE == LIN_FULL) {
                    // FS = F S^T = (I + H)(I + E)^T; Y = Q^T (F S^T)  (column (a,b): dG S F^T = e_a (F S^T)[:,b]^T;
                    // S is symmetric except for plastic iterate bases)
                    T F[9], S[9], FS[9], Y[9];
#pragma unroll
                    for (int a = 0; a < 3; a++)
#pragma unroll
                        for (int b = 0; b < 3; b++) {
                            F[3 * a + b] = H[3 * a + b] + ((a == b) ? T(1) : T(0));
                            S[3 * a + b] = E[3 * b + a] + ((a == b) ? T(1) : T(0));  // S^T
                        }
                    mm3(F, S, FS);
#pragma unroll
                    for (int i = 0; i < 3; i++)
#pragma unroll
                        for (int b = 0; b < 3; b++) Y[3 * i + b] = Q[i] * FS[b] + Q[3 + i] * FS[3 + b] + Q[6 + i] * FS[6 + b];
                    T L[9];
#pragma unroll
                    for (int i = 0; i < 3; i++)
#pragma unroll
                        for (int jj = 0; jj < 3; jj++) L[3 * i + jj] = dlog(lam3[i], lam3[jj]);
                    if (KC) {
                        // compressed tangent of this slot: F = U Sigma V^T (U = eigenvectors of b = F F^T,
                        // sigma_i^2 = beta_i), d^2 psi / dF^2 in the SVD frame = a 3x3 block on the diagonal
                        // entries (psi_ij) and 2x2 blocks [[a, b], [b, a]] on (X_ij, X_ji) (Irving, Teran &
                        // Fedkiw 2004), with g_i = sigma_i psi_i = tp_i for Hencky:
                        //   psi_ij = (2 mu delta_ij + lam) / (sigma_i sigma_j) - delta_ij g_i / sigma_i^2,
                        //   a_ij = (g_i - g_j) / (beta_i - beta_j) = mu L(beta_i, beta_j),
                        //   b_ij = (beta_j a_ij - g_j) / (sigma_i sigma_j);
                        // K : dG = c (C : (dG S)) S, c = dt^2 V / (16 dx^2) (= kscale dt)
                        T U[9], Vm[9], sg[3];
#pragma unroll
                        for (int a = 0; a < 9; a++) U[a] = Q[a];
#pragma unroll
                        for (int i = 0; i < 3; i++) sg[i] = sqrt(T(1) + lam3[i]);
                        const T detU = U[0] * (U[4] * U[8] - U[5] * U[7]) - U[1] * (U[3] * U[8] - U[5] * U[6]) +
                                       U[2] * (U[3] * U[7] - U[4] * U[6]);
                        if (detU < T(0)) { U[2] = -U[2]; U[5] = -U[5]; U[8] = -U[8]; }
#pragma unroll
                        for (int i = 0; i < 3; i++) {  // V[:, i] = F^T U[:, i] / sigma_i
                            const T is = T(1) / sg[i];
#pragma unroll
                            for (int a = 0; a < 3; a++)
                                Vm[3 * a + i] = (F[a] * U[i] + F[3 + a] * U[3 + i] + F[6 + a] * U[6 + i]) * is;
                        }
                        // U D, V D with D = diag(+-1), det D = 1, leave F = U Sigma V^T and C unchanged (the pair
                        // blocks see both X_ij, X_ji scaled by D_i D_j): flip the column pair that makes U's
                        // largest quaternion component w (q (x) i, j, k move x, y, z there), so |w| >= 1/2 and
                        // q_U is stored as (x, y, z) with w = sqrt(1 - x^2 - y^2 - z^2)
                        T qU[4];
                        {
                            rot_quat(U, qU);
                            const T aw = fabs(qU[0]), ax = fabs(qU[1]), ay = fabs(qU[2]), az = fabs(qU[3]);
                            int m = 0;
                            T best = aw;
                            if (ax > best) { m = 1; best = ax; }
                            if (ay > best) { m = 2; best = ay; }
                            if (az > best) m = 3;
                            if (m) {
                                const T d0 = m == 1 ? T(1) : T(-1), d1 = m == 2 ? T(1) : T(-1), d2 = m == 3 ? T(1) : T(-1);
#pragma unroll
                                for (int a = 0; a < 3; a++) {
                                    U[3 * a] *= d0; U[3 * a + 1] *= d1; U[3 * a + 2] *= d2;
                                    Vm[3 * a] *= d0; Vm[3 * a + 1] *= d1; Vm[3 * a + 2] *= d2;
                                }
                                rot_quat(U, qU);
                            }
                            if (qU[0] < T(0)) { qU[1] = -qU[1]; qU[2] = -qU[2]; qU[3] = -qU[3]; }
                        }
                        const T c = sV * T(1.0 / 16.0) * T(g.inv_dx * g.inv_dx) * dt;  // kscale dt
                        // c psi (00 11 22 01 12 02) and c (a, b) of the pairs (0,1) (0,2) (1,2)
                        T ps[6], ab[6];
                        {
                            T psi[9];
#pragma unroll
                            for (int i = 0; i < 3; i++)
#pragma unroll
                                for (int jj = 0; jj < 3; jj++)
                                    psi[3 * i + jj] = ((i == jj ? T(2) * mu : T(0)) + lamL) / (sg[i] * sg[jj]) -
                                                      (i == jj ? tp[i] / (sg[i] * sg[i]) : T(0));
                            ps[0] = c * psi[0]; ps[1] = c * psi[4]; ps[2] = c * psi[8];
                            ps[3] = c * psi[1]; ps[4] = c * psi[5]; ps[5] = c * psi[2];
                        }
                        const int pi_[3] = {0, 0, 1}, pj_[3] = {1, 2, 2};
#pragma unroll
                        for (int pp = 0; pp < 3; pp++) {
                            const int i = pi_[pp], jj = pj_[pp];
                            const T a_ = mu * L[3 * i + jj];
                            const T b_ = ((T(1) + lam3[jj]) * a_ - tp[jj]) / (sg[i] * sg[jj]);
                            ab[2 * pp] = c * a_;
                            ab[2 * pp + 1] = c * b_;
                        }
                        if (PSD) {
                            // S = I: the per-cell PSD projection of K = c C is C's blockwise clamping (amb-6b):
                            // the 3x3 block by its eigenvalues, each [[a, b], [b, a]] by a + b and a - b
                            T Dm[9] = {ps[0], ps[3], ps[5], ps[3], ps[1], ps[4], ps[5], ps[4], ps[2]};
                            T dw[3], DQ[9];
                            sym_eig3(Dm, dw, DQ);
#pragma unroll
                            for (int i = 0; i < 3; i++) dw[i] = dw[i] > T(0) ? dw[i] : T(0);
                            auto dent = [&](int r, int cc) {
                                return DQ[3 * r] * DQ[3 * cc] * dw[0] + DQ[3 * r + 1] * DQ[3 * cc + 1] * dw[1] +
                                       DQ[3 * r + 2] * DQ[3 * cc + 2] * dw[2];
                            };
                            ps[0] = dent(0, 0); ps[1] = dent(1, 1); ps[2] = dent(2, 2);
                            ps[3] = dent(0, 1); ps[4] = dent(1, 2); ps[5] = dent(0, 2);
#pragma unroll
                            for (int pp = 0; pp < 3; pp++) {
                                const T a_ = ab[2 * pp], b_ = ab[2 * pp + 1];
                                const T lp = a_ + b_ > T(0) ? a_ + b_ : T(0), lm = a_ - b_ > T(0) ? a_ - b_ : T(0);
                                ab[2 * pp] = T(0.5) * (lp + lm);
                                ab[2 * pp + 1] = T(0.5) * (lp - lm);
                            }
                        }
                        // W = S V (S symmetric: the elastic base), so K : dG = c U (C : (U^T dG W)) W^T
                        T Wm[9];
#pragma unroll
                        for (int a = 0; a < 3; a++)
#pragma unroll
                            for (int jj = 0; jj < 3; jj++)
                                Wm[3 * a + jj] = S[3 * a] * Vm[jj] + S[3 * a + 1] * Vm[3 + jj] + S[3 * a + 2] * Vm[6 + jj];
                        // the Jacobi diagonal (node phase) reads only K's blocks K[(a,b),(a,e)]:
                        // K[(a,b),(a,e)] = c X_b : C : X_e with X_b = U^T e_a e_b^T W = u_a w_b^T, u_a = U[a][:],
                        // w_b = W[b][:]
                        T *Kr = Ks + j * 45;
#pragma unroll
                        for (int a = 0; a < 3; a++) {
                            T X[3][9];
#pragma unroll
                            for (int b = 0; b < 3; b++)
#pragma unroll
                                for (int i = 0; i < 3; i++)
#pragma unroll
                                    for (int jj = 0; jj < 3; jj++) X[b][3 * i + jj] = U[3 * a + i] * Wm[3 * b + jj];
#pragma unroll
                            for (int b = 0; b < 3; b++)
#pragma unroll
                                for (int e = b; e < 3; e++) {
                                    const T *x = X[b], *y = X[e];
                                    T val = ps[0] * x[0] * y[0] + ps[1] * x[4] * y[4] + ps[2] * x[8] * y[8] +
                                            ps[3] * (x[0] * y[4] + x[4] * y[0]) + ps[4] * (x[4] * y[8] + x[8] * y[4]) +
                                            ps[5] * (x[0] * y[8] + x[8] * y[0]);
#pragma unroll
                                    for (int pp = 0; pp < 3; pp++) {
                                        const int ij = 3 * pi_[pp] + pj_[pp], ji = 3 * pj_[pp] + pi_[pp];
                                        val += ab[2 * pp] * (x[ij] * y[ij] + x[ji] * y[ji]) +
                                               ab[2 * pp + 1] * (x[ij] * y[ji] + x[ji] * y[ij]);
                                    }
                                    Kr[kidx(3 * a + b, 3 * a + e)] += val;
                                }
                        }
                        // the 24 reals: q_U's (x, y, z) (3), W (9, row-major), c psi (6), c (a, b) x 3 (6)
                        // (k_hvp_wz kc_apply2)
                        T kc_[KC_REALS];
                        kc_[0] = qU[1]; kc_[1] = qU[2]; kc_[2] = qU[3];
#pragma unroll
                        for (int e = 0; e < 9; e++) kc_[3 + e] = Wm[e];
#pragma unroll
                        for (int e = 0; e < 6; e++) { kc_[12 + e] = ps[e]; kc_[18 + e] = ab[e]; }
#pragma unroll
                        for (int e = 0; e < KC_REALS; e++) Kout[kc_base + (int64_t)(e >> 1) * 4 * kc_np + 2 * (e & 1)] = kc_[e];
                        kc_done = true;
                    }
                    const T kscale = sV * T(1.0 / 16.0) * T(g.inv_dx * g.inv_dx);
                    T *Kr = Ks + j * 45;
                    if (!KC)  // (KC: the diagonal blocks were assembled above from the compressed form)
#pragma unroll
                    for (int a = 0; a < 3; a++)
#pragma unroll
                        for (int b = 0; b < 3; b++) {
                            // db' = dt (q_a (x) y_b + y_b (x) q_a), q_a[i] = Q[a][i], y_b[i] = Y[i][b]
                            T Dp[9];
                            T trD = T(0);
#pragma unroll
                            for (int i = 0; i < 3; i++)
#pragma unroll
                                for (int jj = 0; jj < 3; jj++) {
                                    T dbp = dt * (Q[3 * a + i] * Y[3 * jj + b] + Y[3 * i + b] * Q[3 * a + jj]);
                                    Dp[3 * i + jj] = L[3 * i + jj] * dbp;
                                }
                            trD = Dp[0] + Dp[4] + Dp[8];
                            // dtau' = mu D' + lam/2 tr(D') I ; dtau = Q dtau' Q^T
                            T dtp[9];
#pragma unroll
                            for (int i = 0; i < 9; i++) dtp[i] = mu * Dp[i] + ((i % 4 == 0) ? T(0.5) * lamL * trD : T(0));
                            T tmp[9], dtau[9];
#pragma unroll
                            for (int i = 0; i < 3; i++)
#pragma unroll
                                for (int jj = 0; jj < 3; jj++)
                                    tmp[3 * i + jj] = Q[3 * i] * dtp[jj] + Q[3 * i + 1] * dtp[3 + jj] + Q[3 * i + 2] * dtp[6 + jj];
#pragma unroll
                            for (int i = 0; i < 3; i++)
#pragma unroll
                                for (int jj = 0; jj < 3; jj++)
                                    dtau[3 * i + jj] = tmp[3 * i] * Q[3 * jj] + tmp[3 * i + 1] * Q[3 * jj + 1] + tmp[3 * i + 2] * Q[3 * jj + 2];
                            // column (a,b): dtau A^{-T} - dt (tau A^{-T}) e_b (x) e_a^T A^{-T}
                            const int cidx = 3 * a + b;
#pragma unroll
                            for (int i = 0; i < 3; i++)
#pragma unroll
                                for (int jj = 0; jj < 3; jj++) {
                                    T r1 = dtau[3 * i] * AiT[jj] + dtau[3 * i + 1] * AiT[3 + jj] + dtau[3 * i + 2] * AiT[6 + jj];
                                    T r2 = -dt * TA[3 * i + b] * AiT[3 * a + jj];
                                    T val = kscale * (r1 + r2);
                                    const int r = 3 * i + jj;
                                    if (r == cidx) Kr[kidx(r, r)] += val;
                                    else if (r < cidx) Kr[kidx(r, cidx)] += T(0.5) * val;
                                    else Kr[kidx(cidx, r)] += T(0.5) * val;
                                }
                        }
                }
            }
            if (MODE != LIN_ENERGY) {
#pragma unroll
                for (int a = 0; a < 9; a++) Pg[l * 9 + a] = Pc[a] * q;  // fold grad w scale
            }
            if (KC && !kc_done)  // no occupied slot (a zero-mass stencil cell, amb-10): zero tangent
                for (int e = 0; e < KC_REALS; e++) Kout[kc_base + (int64_t)(e >> 1) * 4 * kc_np + 2 * (e & 1)] = T(0);
        }
    }
    __syncthreads();
    if (PSD && MODE == LIN_FULL && has) {  // per-cell PSD projection before the K write and the diagonal
        if (!(KC) && tid < nc && clocal[cs + tid] != 0xFF)
            psd_project45<T>(Ks + tid * 45);  // fp64: spills, acceptable
        __syncthreads();
    }
    if (MODE == LIN_FULL && has) {  // tile's tangent block, permuted into the chunked (coalesced) layout
        const int64_t base = kstart[t];
        const int n = ncell[t];  // real cells come first in the compact run
        // slot of each cell: kz == 1 (k_hvp_wz lanes): the rank of its kz_key among the tile's cells;
        // kz == 3 (k_hvp_wh): its rank in the natural compact order
        if (tid < n) {
            int sl = tid;
            if (kz == 1) {
                const int key = kz_key(clocal[cs + tid]);
                sl = 0;
                for (int j = 0; j < n; j++) sl += kz_key(clocal[cs + j]) < key;
            }
            zslot[tid] = sl;
        }
        __syncthreads();
        if (KC) {
            // written by the cell phase (pair layout)
        } else {
            for (int i = tid; i < n * 45; i += blockDim.x) Kout[k_off<T>(base, n, zslot[i / 45], i % 45)] = Ks[i];
        }
    }
    // ---- node phase -----------------------------------------------------------------------
    for (int h = tid; h < 125; h += blockDim.x) {
        int hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        bool owned = hx < 4 && hy < 4 && hz < 4;
        bool interior = hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3;
        T f[3] = {0, 0, 0}, d[3] = {0, 0, 0};
        bool any = false;
        if (has && MODE != LIN_ENERGY) {
#pragma unroll
            for (int o = 0; o < 8; o++) {
                int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
                int cx = hx - ox, cy = hy - oy, cz = hz - oz;
                if (cx < 0 || cy < 0 || cz < 0 || cx > 3 || cy > 3 || cz > 3) continue;
                int l = local_id(cx, cy, cz);
                int jj = cslot[l];
                if (jj < 0 || clocal[cs + jj] == 0xFF) continue;
                any = true;
                T s[3] = {ox ? T(1) : T(-1), oy ? T(1) : T(-1), oz ? T(1) : T(-1)};
                const T *P = Pg + l * 9;
#pragma unroll
                for (int a = 0; a < 3; a++) f[a] += P[3 * a] * s[0] + P[3 * a + 1] * s[1] + P[3 * a + 2] * s[2];
                if (MODE == LIN_FULL) {
                    const T *Kr = Ks + jj * 45;
#pragma unroll
                    for (int a = 0; a < 3; a++) {
                        T acc = T(0);
#pragma unroll
                        for (int b = 0; b < 3; b++)
#pragma unroll
                            for (int e = 0; e < 3; e++) {
                                int r = 3 * a + b, c = 3 * a + e;
                                T kv = r <= c ? Kr[kidx(r, c)] : Kr[kidx(c, r)];
                                acc += s[b] * s[e] * kv;
                            }
                        d[a] += acc;
                    }
                }
            }
        }
        int64_t n = (owned || has) ? halo_node(t, nplus, h) : -1;
        DASSERT(n < (int64_t)gridDim.x * 64);
        if (n >= 0) {
            if (owned) {
                T m = nmass[n];
                if (m > T(0)) {
                    vec4<T> vv = vh[h], vt = vhat[n];
                    T dv0 = vv.x - vt.x, dv1 = vv.y - vt.y, dv2 = vv.z - vt.z;
                    e_loc += 0.5 * (double)(m * (dv0 * dv0 + dv1 * dv1 + dv2 * dv2));
                    f[0] += m * dv0; f[1] += m * dv1; f[2] += m * dv2;
                    d[0] += m; d[1] += m; d[2] += m;
                    any = true;
                }
            }
            if (MODE != LIN_ENERGY && any) {
                if (interior || !has) {
                    // exclusive: all 8 cells of an interior node lie in this tile; a tile without
                    // cells contributes only the mass terms of its owned nodes
                    if (interior) {
                        grad[n] = mk4<T>(f[0], f[1], f[2], T(0));
                        if (MODE == LIN_FULL) diag[n] = mk4<T>(d[0], d[1], d[2], T(0));
                    } else {
                        atomic_add3<T>(grad + n, f[0], f[1], f[2]);
                        if (MODE == LIN_FULL) atomic_add3<T>(diag + n, d[0], d[1], d[2]);
                    }
                } else {
                    atomic_add3<T>(grad + n, f[0], f[1], f[2]);
                    if (MODE == LIN_FULL) atomic_add3<T>(diag + n, d[0], d[1], d[2]);
                }
            }
        }
    }
    block_add(e_loc, sc->energy);
}

// =============================================================================================
// Explicit integration (Eq. explicitforce, Alg. 3 lines 1-3):
//   f_i = - sum_c sum_k V_ck tau_ck grad w_ic ,   v_i^{n+1} = v_i^n + dt (g + f_i / m_i)  (gravity amb-4)
// on the same tiles: per cell Pc = sum_k V_ck tau_ck (the quadrature stress content of P2Q), scattered
// to the 8 corners with grad w_ic = s_ic / (4 dx); interior nodes stored, face nodes atomically added.
// =============================================================================================
template <class T>
__global__ void __launch_bounds__(128) k_explicit_force(GridP g, int nmat, const int *__restrict__ nplus,
                                                        const int *__restrict__ cstart,
                                                        const uint8_t *__restrict__ clocal,
                                                        const int *__restrict__ hascells, const T *__restrict__ qslot,
                                                        vec4<T> *__restrict__ f) {
    __shared__ T Pg[64 * 9];
    __shared__ int cslot[64];
    const int t = blockIdx.x, tid = threadIdx.x;
    const int has = hascells[t];
    if (!has) return;
    const int cs = cstart[t], nc = cstart[t + 1] - cs;
    if (tid < 64) cslot[tid] = -1;
    __syncthreads();
    const T q = T(0.25 * g.inv_dx);
    if (tid < nc) {
        const int l = clocal[cs + tid];
        if (l != 0xFF) {
            cslot[l] = tid;
            T P[6] = {0, 0, 0, 0, 0, 0};
            for (int k = 0; k < nmat; k++) {
                const T *sl = qslot + ((int64_t)(cs + tid) * nmat + k) * 16;
                const T V = sl[0];
#pragma unroll
                for (int a = 0; a < 6; a++) P[a] += V * sl[7 + a];  // V_ck tau_ck (xx yy zz xy yz xz)
            }
            const T full[9] = {P[0], P[3], P[5], P[3], P[1], P[4], P[5], P[4], P[2]};
#pragma unroll
            for (int a = 0; a < 9; a++) Pg[l * 9 + a] = -full[a] * q;  // f = -V tau grad w
        }
    }
    __syncthreads();
    if (tid < 125) {
        const int h = tid, hx = h / 25, hy = (h / 5) % 5, hz = h % 5;
        const bool interior = hx >= 1 && hx <= 3 && hy >= 1 && hy <= 3 && hz >= 1 && hz <= 3;
        T fv[3] = {0, 0, 0};
        bool any = false;
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
            const int cx = hx - ox, cy = hy - oy, cz = hz - oz;
            if (cx < 0 || cy < 0 || cz < 0 || cx > 3 || cy > 3 || cz > 3) continue;
            const int l = local_id(cx, cy, cz);
            if (cslot[l] < 0) continue;
            any = true;
            const T s0 = ox ? T(1) : T(-1), s1 = oy ? T(1) : T(-1), s2 = oz ? T(1) : T(-1);
            const T *P = Pg + l * 9;
#pragma unroll
            for (int a = 0; a < 3; a++) fv[a] += P[3 * a] * s0 + P[3 * a + 1] * s1 + P[3 * a + 2] * s2;
        }
        const int64_t n = halo_node(t, nplus, h);
        if (any && n >= 0) {
            if (interior) f[n] = mk4<T>(fv[0], fv[1], fv[2], T(0));
            else atomic_add3<T>(f + n, fv[0], fv[1], fv[2]);
        }
    }
}

// v^{n+1} = vhat + dt f / m on free nodes (vhat = v^n + dt g); prescribed nodes keep their value
template <class T>
__global__ void k_explicit_update(int64_t n, const int *__restrict__ list, const uint8_t *__restrict__ flag,
                                  const vec4<T> *__restrict__ vhat, const T *__restrict__ m,
                                  const vec4<T> *__restrict__ f, T dt, vec4<T> *__restrict__ v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ti = list[i];
    if (flag[ti] != 1) return;
    const vec4<T> vh = vhat[ti], fv = f[ti];
    const T s = dt / m[ti];
    v[ti] = mk4<T>(vh.x + s * fv.x, vh.y + s * fv.y, vh.z + s * fv.z, T(0));
}

// =============================================================================================
// a7: Jacobi-PCG vector kernels (fp64 accumulation of every dot product)
// slot j: rz_j = r_j.z_j, rr_j = r_j.r_j, pHp_j = p_j.H p_j
// =============================================================================================
// ---- PCG on the compact list of active nodes (i -> tile-dense slot list[i]) ---------------------
// x, r and invD are compact over the active nodes and stored component-major (SoA): component c of
// node i at a[c * S + i], S = the active-node count rounded up to 4, 12 bytes per node in fp32 instead
// of a 16-byte vec4; p and Hp stay tile-dense vec4 because the HVP gathers and scatters them by tile.
// Prescribed DOFs have invD = 0 (that is the free mask) and r = p = 0.  own (slab ranks only, else
// nullptr) weights each node's dot-product terms so shared interface nodes count once.

// 4 consecutive reals (16-byte aligned)
template <class T> struct R4 { T v[4]; };
template <class T> __device__ __forceinline__ R4<T> ld4(const T *p);
template <> __device__ __forceinline__ R4<float> ld4<float>(const float *p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    return R4<float>{{a.x, a.y, a.z, a.w}};
}
template <> __device__ __forceinline__ R4<double> ld4<double>(const double *p) {
    const double2 a = reinterpret_cast<const double2 *>(p)[0], b = reinterpret_cast<const double2 *>(p)[1];
    return R4<double>{{a.x, a.y, b.x, b.y}};
}
template <class T> __device__ __forceinline__ void st4(T *p, const T v[4]);
template <> __device__ __forceinline__ void st4<float>(float *p, const float v[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <> __device__ __forceinline__ void st4<double>(double *p, const double v[4]) {
    reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
}
inline int64_t soa_stride(int64_t n) { return (n + 3) & ~(int64_t)3; }

// r = -g, invD = 1/D on free DOFs; z = invD r; p = z; x = 0; slot[0] = (r.z, r.r)
template <class T>
__global__ void __launch_bounds__(256) k_pcg_init(int64_t n, int64_t S, const int *__restrict__ list,
                                                  const uint8_t *__restrict__ flag, const uint8_t *__restrict__ own,
                                                  const vec4<T> *__restrict__ g,
                                                  const vec4<T> *__restrict__ D, T *__restrict__ invD,
                                                  T *__restrict__ r, vec4<T> *__restrict__ p,
                                                  T *__restrict__ x, CGSlot *slot, bool zform) {
    T rz = 0, rr = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
        T rv[3] = {0, 0, 0}, iv[3] = {0, 0, 0};
        if (i < n) {
            const int ti = list[i];
            if (flag[ti] == 1) {
                const vec4<T> gv = g[ti], dv = D[ti];
                const T w = own ? T(own[ti]) : T(1);
                iv[0] = T(1) / dv.x; iv[1] = T(1) / dv.y; iv[2] = T(1) / dv.z;
                rv[0] = -gv.x; rv[1] = -gv.y; rv[2] = -gv.z;
                const T z0 = rv[0] * iv[0], z1 = rv[1] * iv[1], z2 = rv[2] * iv[2];
                rz += w * (rv[0] * z0 + rv[1] * z1 + rv[2] * z2);
                rr += w * (rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
                p[ti] = mk4<T>(z0, z1, z2, T(0));
            }
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
            invD[c * S + i] = iv[c];
            r[c * S + i] = zform ? rv[c] * iv[c] : rv[c];  // zform: the buffer holds z = D^-1 r
            x[c * S + i] = T(0);
        }
    }
    block_add((double)rz, slot[0].rz);
    block_add((double)rr, slot[0].rr);
}

// Scalars of CG iteration j, read once per CTA: rr_j, pHp_j, rz_j, rz_{j+1}, rr_{j+1} (striped sums).
struct CGScal {
    double rr, pHp, rz, rz1, rr1;
};
__device__ __forceinline__ CGScal cg_scalars(const CGSlot *slot, int j, bool next) {
    __shared__ CGScal s_;
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        double a = warp_sum(slot[j].rr[l]), b = warp_sum(slot[j].pHp[l]), c = warp_sum(slot[j].rz[l]);
        double d = next ? warp_sum(slot[j + 1].rz[l]) : 0.0, e = next ? warp_sum(slot[j + 1].rr[l]) : 0.0;
        if (l == 0) s_ = CGScal{a, b, c, d, e};
    }
    __syncthreads();
    return s_;
}

// a group = 4 consecutive compact nodes i0..i0+3: their list entries (-1 past n)
constexpr int PCG_U = 1;  // groups per thread per pass
__device__ __forceinline__ void grp_list(const int *__restrict__ list, int64_t i0, int64_t n, int li[4]) {
    if (i0 + 4 <= n) {
        const int4 l = *reinterpret_cast<const int4 *>(list + i0);
        li[0] = l.x; li[1] = l.y; li[2] = l.z; li[3] = l.w;
    } else {
#pragma unroll
        for (int e = 0; e < 4; e++) li[e] = i0 + e < n ? list[i0 + e] : -1;
    }
}

// k_pcg_update1: r -= alpha Hp ; slot[j+1] = (r.invD r, r.r) ; Hp := 0 for the next HVP's atomics.
// k_pcg_update2: x += alpha_j p_j ; then (unless converged) p = invD r + beta p, beta = rz_{j+1} / rz_j.
// (x is updated in update2, which reads p anyway: one fewer pass over p.)
// Persistent: one CTA wave (SMs x 8 CTAs of 256), the CG scalars read once per CTA; each thread takes
// groups of 4 consecutive nodes (16-byte loads of every SoA component and of the list), every
// independent load issued before the dependent tile-dense one (list -> Hp / p).  Bytes per node (fp32):
// update1 72 (invD 12, r 12 + 12, Hp 16 + 16, list 4), update2 84 (vec4 x / r / invD: 84 and 100).
// A warp-interleaved mapping (lane l: nodes l + 32 e, scalar component loads) measured slower.
// One node per thread (~9000 CTAs) was 3x slower: each CTA's two striped fp64 atomics serialised on
// the slot's cache lines (ncu: long scoreboard 72 %, barrier 20 %; 104 us vs 34 us live at cfg4).
template <class T, int U>
__global__ void __launch_bounds__(256) k_pcg_update1(int64_t n, int64_t S, const int *__restrict__ list, int j,
                                                      double thr, const T *__restrict__ invD,
                                                      const vec4<T> *__restrict__ p, vec4<T> *__restrict__ Hp,
                                                      T *__restrict__ x, T *__restrict__ r,
                                                      const uint8_t *__restrict__ own, CGSlot *slot, DevScalars *sc) {
    pdl_trigger();
    pdl_wait();
    const CGScal cs = cg_scalars(slot, j, false);
    const int done = sc->cg_done_iter;
    if ((done >= 0 && done <= j) || (j > 0 && cs.rr <= thr)) return;
    const int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    const int64_t NG = (n + 3) >> 2;
    if (!(cs.pHp > 0.0)) {
        if (j == 0)
            for (int64_t i = g0; i < n; i += gs) {
                const vec4<T> pv = p[list[i]];
                x[i] = pv.x; x[S + i] = pv.y; x[2 * S + i] = pv.z;
            }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sc->neg_curv = 1;
            sc->cg_done_iter = j + 1;
        }
        return;
    }
    const T alpha = T(cs.rz / cs.pHp);
    T rz = 0, rr = 0;
    for (int64_t b = g0; b < NG; b += gs * U) {
        int li[U][4];
        T iv[U][3][4], rv[U][3][4];
        vec4<T> hv[U][4];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i0 = 4 * (b + u * gs);
            if (i0 >= n) { li[u][0] = li[u][1] = li[u][2] = li[u][3] = -1; continue; }
            grp_list(list, i0, n, li[u]);
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const R4<T> a = ld4<T>(invD + c * S + i0), q = ld4<T>(r + c * S + i0);
#pragma unroll
                for (int e = 0; e < 4; e++) { iv[u][c][e] = a.v[e]; rv[u][c][e] = q.v[e]; }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int e = 0; e < 4; e++)
                if (li[u][e] >= 0) hv[u][e] = Hp[li[u][e]];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i0 = 4 * (b + u * gs);
            if (i0 >= n) continue;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (li[u][e] < 0) continue;
                Hp[li[u][e]] = mk4<T>(0, 0, 0, 0);
                const T aw = iv[u][0][e] != T(0) ? alpha : T(0);  // prescribed DOFs keep r = 0
                rv[u][0][e] -= aw * hv[u][e].x; rv[u][1][e] -= aw * hv[u][e].y; rv[u][2][e] -= aw * hv[u][e].z;
                const T w = own ? T(own[li[u][e]]) : T(1);
                rz += w * (rv[u][0][e] * rv[u][0][e] * iv[u][0][e] + rv[u][1][e] * rv[u][1][e] * iv[u][1][e] +
                           rv[u][2][e] * rv[u][2][e] * iv[u][2][e]);
                rr += w * (rv[u][0][e] * rv[u][0][e] + rv[u][1][e] * rv[u][1][e] + rv[u][2][e] * rv[u][2][e]);
            }
#pragma unroll
            for (int c = 0; c < 3; c++) st4<T>(r + c * S + i0, rv[u][c]);  // S padding absorbs the tail
        }
    }
    block_add((double)rz, slot[j + 1].rz);
    block_add((double)rr, slot[j + 1].rr);
}

template <class T, int U>
__global__ void __launch_bounds__(256) k_pcg_update2(int64_t n, int64_t S, const int *__restrict__ list, int j,
                                                      double thr, const T *__restrict__ invD,
                                                      const T *__restrict__ r, vec4<T> *__restrict__ p,
                                                      T *__restrict__ x, const CGSlot *slot, const DevScalars *sc) {
    pdl_trigger();
    pdl_wait();
    const CGScal cs = cg_scalars(slot, j, true);
    const int done = sc->cg_done_iter;
    if ((done >= 0 && done <= j + 1) || (j > 0 && cs.rr <= thr)) return;
    const T alpha = T(cs.rz / cs.pHp);
    const bool more = cs.rr1 > thr;
    const T beta = more ? T(cs.rz1 / cs.rz) : T(0);
    const int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    const int64_t NG = (n + 3) >> 2;
    for (int64_t b = g0; b < NG; b += gs * U) {
        int li[U][4];
        T xv[U][3][4], rv[U][3][4], iv[U][3][4];
        vec4<T> pv[U][4];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i0 = 4 * (b + u * gs);
            if (i0 >= n) { li[u][0] = li[u][1] = li[u][2] = li[u][3] = -1; continue; }
            grp_list(list, i0, n, li[u]);
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const R4<T> a = ld4<T>(x + c * S + i0);
#pragma unroll
                for (int e = 0; e < 4; e++) xv[u][c][e] = a.v[e];
                if (more) {
                    const R4<T> q = ld4<T>(r + c * S + i0), d = ld4<T>(invD + c * S + i0);
#pragma unroll
                    for (int e = 0; e < 4; e++) { rv[u][c][e] = q.v[e]; iv[u][c][e] = d.v[e]; }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int e = 0; e < 4; e++)
                if (li[u][e] >= 0) pv[u][e] = p[li[u][e]];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i0 = 4 * (b + u * gs);
            if (i0 >= n) continue;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (li[u][e] < 0) continue;
                xv[u][0][e] += alpha * pv[u][e].x; xv[u][1][e] += alpha * pv[u][e].y; xv[u][2][e] += alpha * pv[u][e].z;
                if (more)
                    p[li[u][e]] = mk4<T>(rv[u][0][e] * iv[u][0][e] + beta * pv[u][e].x,
                                         rv[u][1][e] * iv[u][1][e] + beta * pv[u][e].y,
                                         rv[u][2][e] * iv[u][2][e] + beta * pv[u][e].z, T(0));
            }
#pragma unroll
            for (int c = 0; c < 3; c++) st4<T>(x + c * S + i0, xv[u][c]);
        }
    }
}

// Warp-interleaved variants (MPL_PCG_MAP=warp): a warp takes chunks of 32 PCG_E compact nodes, lane l
// the nodes l + 32 e, so every SoA component load, list load and tile-dense p / Hp access of one
// instruction is contiguous across the warp (the group mapping above writes p / Hp at a 64-byte lane
// stride).  Full chunks run without per-node bounds checks.
constexpr int PCG_E = 4;  // nodes per lane per chunk (2 with 4 CTAs per SM measured slower: cfg4 step 65.2 vs 59.1 ms)
template <class T, int E = PCG_E, int MB = 2, bool ZF = false>
__global__ void __launch_bounds__(256, MB) k_pcg_update1w(int64_t n, int64_t S, const int *__restrict__ list, int j,
                                                         double thr, const T *__restrict__ invD,
                                                         const vec4<T> *__restrict__ p, vec4<T> *__restrict__ Hp,
                                                         T *__restrict__ x, T *__restrict__ r,
                                                         const uint8_t *__restrict__ own, CGSlot *slot,
                                                         DevScalars *sc, const int *__restrict__ jdev = nullptr) {
    pdl_trigger();
    pdl_wait();
    if (jdev) {  // graph-captured PCG: iteration index and threshold from device memory
        j = *jdev;
        thr = sc->cg_thr;
    }
    const CGScal cs = cg_scalars(slot, j, false);
    const int done = sc->cg_done_iter;
    if ((done >= 0 && done <= j) || (j > 0 && cs.rr <= thr)) return;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (!(cs.pHp > 0.0)) {
        if (j == 0)
            for (int64_t i = w0 * 32 + lane; i < n; i += nw * 32) {
                const vec4<T> pv = p[list[i]];
                x[i] = pv.x; x[S + i] = pv.y; x[2 * S + i] = pv.z;
            }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sc->neg_curv = 1;
            sc->cg_done_iter = j + 1;
        }
        return;
    }
    const T alpha = T(cs.rz / cs.pHp);
    T rz = 0, rr = 0;
    auto chunk = [&](int64_t base, auto full) {
        constexpr bool FULL = decltype(full)::value;
        int li[E];
        T iv[E][3], rv[E][3];
        vec4<T> hv[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int64_t i = base + 32 * e + lane;
            if (FULL || i < n) {
                li[e] = list[i];
#pragma unroll
                for (int c = 0; c < 3; c++) { iv[e][c] = invD[c * S + i]; rv[e][c] = r[c * S + i]; }
            } else {
                li[e] = -1;
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++)
            if (FULL || li[e] >= 0) hv[e] = Hp[li[e]];
#pragma unroll
        for (int e = 0; e < E; e++) {
            if (!FULL && li[e] < 0) continue;
            const int64_t i = base + 32 * e + lane;
            Hp[li[e]] = mk4<T>(0, 0, 0, 0);
            const T w = own ? T(own[li[e]]) : T(1);
            if (ZF) {  // the buffer holds z = D^-1 r: z -= (alpha D^-1) Hp; prescribed DOFs have D^-1 = 0, z = 0
                const T hc[3] = {hv[e].x, hv[e].y, hv[e].z};
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    const T zc = rv[e][c] - (alpha * iv[e][c]) * hc[c];
                    r[c * S + i] = zc;
                    const T rc = iv[e][c] != T(0) ? __fdividef(zc, iv[e][c]) : T(0);  // r = D z
                    rz += w * (rc * zc);
                    rr += w * (rc * rc);
                }
                continue;
            }
            const T aw = iv[e][0] != T(0) ? alpha : T(0);  // prescribed DOFs keep r = 0
            rv[e][0] -= aw * hv[e].x; rv[e][1] -= aw * hv[e].y; rv[e][2] -= aw * hv[e].z;
#pragma unroll
            for (int c = 0; c < 3; c++) r[c * S + i] = rv[e][c];
            rz += w * (rv[e][0] * rv[e][0] * iv[e][0] + rv[e][1] * rv[e][1] * iv[e][1] + rv[e][2] * rv[e][2] * iv[e][2]);
            rr += w * (rv[e][0] * rv[e][0] + rv[e][1] * rv[e][1] + rv[e][2] * rv[e][2]);
        }
    };
    for (int64_t ch = w0; ch * 32 * E < n; ch += nw) {
        const int64_t base = ch * 32 * E;
        if (base + 32 * E <= n) chunk(base, std::true_type{});
        else chunk(base, std::false_type{});
    }
    block_add((double)rz, slot[j + 1].rz);
    block_add((double)rr, slot[j + 1].rr);
}

template <class T, int E = PCG_E, int MB = 2, bool ZF = false>
__global__ void __launch_bounds__(256, MB) k_pcg_update2w(int64_t n, int64_t S, const int *__restrict__ list, int j,
                                                         double thr, const T *__restrict__ invD,
                                                         const T *__restrict__ r, vec4<T> *__restrict__ p,
                                                         T *__restrict__ x, const CGSlot *slot, const DevScalars *sc,
                                                         const int *__restrict__ jdev = nullptr,
                                                         int *__restrict__ jout = nullptr) {
    pdl_trigger();
    pdl_wait();
    if (jdev) {  // graph-captured PCG: this iteration's index; the next iteration's kernels read jout
        j = *jdev;
        thr = sc->cg_thr;
        if (blockIdx.x == 0 && threadIdx.x == 0) *jout = j + 1;
    }
    const CGScal cs = cg_scalars(slot, j, true);
    const int done = sc->cg_done_iter;
    if ((done >= 0 && done <= j + 1) || (j > 0 && cs.rr <= thr)) return;
    const T alpha = T(cs.rz / cs.pHp);
    const bool more = cs.rr1 > thr;
    const T beta = more ? T(cs.rz1 / cs.rz) : T(0);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    auto chunk = [&](int64_t base, auto full) {
        constexpr bool FULL = decltype(full)::value;
        int li[E];
        T xv[E][3], rv[E][3], iv[E][3];
        vec4<T> pv[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int64_t i = base + 32 * e + lane;
            if (FULL || i < n) {
                li[e] = list[i];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    xv[e][c] = x[c * S + i];
                    if (more) {
                        rv[e][c] = r[c * S + i];
                        iv[e][c] = ZF ? T(1) : invD[c * S + i];  // ZF: r holds z = D^-1 r already
                    }
                }
            } else {
                li[e] = -1;
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++)
            if (FULL || li[e] >= 0) pv[e] = p[li[e]];
#pragma unroll
        for (int e = 0; e < E; e++) {
            if (!FULL && li[e] < 0) continue;
            const int64_t i = base + 32 * e + lane;
            x[i] = xv[e][0] + alpha * pv[e].x;
            x[S + i] = xv[e][1] + alpha * pv[e].y;
            x[2 * S + i] = xv[e][2] + alpha * pv[e].z;
            if (more)
                p[li[e]] = mk4<T>(rv[e][0] * iv[e][0] + beta * pv[e].x, rv[e][1] * iv[e][1] + beta * pv[e].y,
                                  rv[e][2] * iv[e][2] + beta * pv[e].z, T(0));
        }
    };
    for (int64_t ch = w0; ch * 32 * E < n; ch += nw) {
        const int64_t base = ch * 32 * E;
        if (base + 32 * E <= n) chunk(base, std::true_type{});
        else chunk(base, std::false_type{});
    }
}

// ---- single-reduction Jacobi-PCG (Chronopoulos & Gear's recurrence; MPL_PCG=cg1, the default) ------
// Mathematically the Hestenes-Stiefel PCG of the oracle (amb-7, amb-8): the matrix-vector product is
// applied to the preconditioned residual u = D^-1 r instead of to p, and s = H p is carried by the
// recurrence s_j = w_j + beta_j s_{j-1} (w_j = H u_j), so every scalar of iteration j is known once
// its HVP has run:
//   gamma_j = r_j . u_j (vector kernel j-1),  delta_j = u_j . H u_j (HVP epilogue, quadratic form),
//   beta_j = gamma_j / gamma_{j-1},  eta_j = delta_j - beta_j gamma_j / alpha_{j-1}  (= p_j . H p_j),
//   alpha_j = gamma_j / eta_j;  eta_j <= 0: negative curvature (iteration 0 returns u_0 = z_0).
// One vector kernel per iteration instead of two, and on slab ranks one allreduce (gamma, r.r, delta)
// instead of two.  u (the HVP input) and w (its output) are tile-dense; x, r, p, s, 1/D compact SoA.
// Per node (fp32): reads r, 1/D, p, s, x (60 B), w (16), list (4); writes r, p, s, x (48), u (16),
// w := 0 (16) for the next HVP's atomics.
template <class T, int E>
__global__ void __launch_bounds__(256, 2) k_pcg_cg1(int64_t n, int64_t S, const int *__restrict__ list, int j,
                                                    double thr, const T *__restrict__ invD, vec4<T> *__restrict__ u,
                                                    vec4<T> *__restrict__ w, T *__restrict__ x, T *__restrict__ r,
                                                    T *__restrict__ p, T *__restrict__ s_,
                                                    const uint8_t *__restrict__ own, CGSlot *slot, DevScalars *sc) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh_[4];
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        const double gam = warp_sum(slot[j].rz[l]), rr = warp_sum(slot[j].rr[l]), del = warp_sum(slot[j].pHp[l]);
        const double gam0 = j > 0 ? warp_sum(slot[j - 1].rz[l]) : 0.0;
        if (l == 0) { sh_[0] = gam; sh_[1] = rr; sh_[2] = del; sh_[3] = gam0; }
    }
    __syncthreads();
    const double gam = sh_[0], rr = sh_[1], del = sh_[2], gam0 = sh_[3];
    const int done = sc->cg_done_iter;
    if ((done >= 0 && done <= j) || (j > 0 && rr <= thr)) return;
    const double beta_d = j > 0 ? gam / gam0 : 0.0;
    const double eta = del - (j > 0 ? beta_d * gam / slot[j - 1].alpha : 0.0);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (!(eta > 0.0)) {  // negative curvature: stop; at j == 0 the step is u_0 = D^-1 r_0 (= z_0)
        if (j == 0)
            for (int64_t i = w0 * 32 + lane; i < n; i += nw * 32)
#pragma unroll
                for (int c = 0; c < 3; c++) x[c * S + i] = invD[c * S + i] * r[c * S + i];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sc->neg_curv = 1;
            sc->cg_done_iter = j + 1;
        }
        return;
    }
    const double alpha_d = gam / eta;
    if (blockIdx.x == 0 && threadIdx.x == 0) slot[j].alpha = alpha_d;
    const T alpha = T(alpha_d), beta = T(beta_d);
    T gsum = 0, rsum = 0;
    auto chunk = [&](int64_t base, auto full) {
        constexpr bool FULL = decltype(full)::value;
        int li[E];
        T iv[E][3], rv[E][3], pv[E][3], sv[E][3], xv[E][3];
        vec4<T> wv[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int64_t i = base + 32 * e + lane;
            if (FULL || i < n) {
                li[e] = list[i];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    iv[e][c] = invD[c * S + i]; rv[e][c] = r[c * S + i]; pv[e][c] = p[c * S + i];
                    sv[e][c] = s_[c * S + i]; xv[e][c] = x[c * S + i];
                }
            } else {
                li[e] = -1;
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++)
            if (FULL || li[e] >= 0) wv[e] = w[li[e]];
#pragma unroll
        for (int e = 0; e < E; e++) {
            if (!FULL && li[e] < 0) continue;
            const int64_t i = base + 32 * e + lane;
            const T wc[3] = {wv[e].x, wv[e].y, wv[e].z};
            T un[3];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                // prescribed DOFs (1/D = 0): r, u, p, s stay 0 (the Hessian is projected onto free DOFs)
                const T fr = iv[e][c] != T(0) ? T(1) : T(0);
                const T pn = iv[e][c] * rv[e][c] + beta * pv[e][c];
                const T sn = fr * (wc[c] + beta * sv[e][c]);
                xv[e][c] += alpha * pn;
                rv[e][c] -= alpha * sn;
                un[c] = iv[e][c] * rv[e][c];
                p[c * S + i] = pn;
                s_[c * S + i] = sn;
                x[c * S + i] = xv[e][c];
                r[c * S + i] = rv[e][c];
            }
            u[li[e]] = mk4<T>(un[0], un[1], un[2], T(0));
            w[li[e]] = mk4<T>(0, 0, 0, 0);
            const T ow = own ? T(own[li[e]]) : T(1);
            gsum += ow * (rv[e][0] * un[0] + rv[e][1] * un[1] + rv[e][2] * un[2]);
            rsum += ow * (rv[e][0] * rv[e][0] + rv[e][1] * rv[e][1] + rv[e][2] * rv[e][2]);
        }
    };
    for (int64_t ch = w0; ch * 32 * E < n; ch += nw) {
        const int64_t base = ch * 32 * E;
        if (base + 32 * E <= n) chunk(base, std::true_type{});
        else chunk(base, std::false_type{});
    }
    block_add((double)gsum, slot[j + 1].rz);
    block_add((double)rsum, slot[j + 1].rr);
}

// g . x over free DOFs (g tile-dense, x compact SoA)
template <class T>
__global__ void k_dot_gx(int64_t n, int64_t S, const int *__restrict__ list, const uint8_t *__restrict__ flag,
                         const uint8_t *__restrict__ own, const vec4<T> *__restrict__ g, const T *__restrict__ x,
                         double *out) {
    double s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int ti = list[i];
        if (flag[ti] != 1 || !own[ti]) continue;
        const vec4<T> a = g[ti];
        s += (double)(a.x * x[i] + a.y * x[S + i] + a.z * x[2 * S + i]);
    }
    block_add(s, out);
}

// vt = v + alpha x on free DOFs (vt pre-filled with v)
template <class T>
__global__ void k_axpy_compact(int64_t n, int64_t S, const int *__restrict__ list, const uint8_t *__restrict__ flag,
                               T alpha, const vec4<T> *__restrict__ v, const T *__restrict__ x,
                               vec4<T> *__restrict__ vt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int ti = list[i];
        if (flag[ti] != 1) continue;
        vec4<T> a = v[ti];
        a.x += alpha * x[i]; a.y += alpha * x[S + i]; a.z += alpha * x[2 * S + i];
        vt[ti] = a;
    }
}

// HVP wrapper used inside PCG: skips work once converged
// graph-captured PCG: iteration counter and threshold of a Newton iteration's solve
__global__ void k_set_cg(DevScalars *sc, double thr) {
    sc->cg_j[0] = 0;
    sc->cg_j[1] = 0;
    sc->cg_thr = thr;
}

template <class T>
__global__ void k_zero4(int64_t N, vec4<T> *a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = mk4<T>(0, 0, 0, 0);
}

// g . x over free nodes
template <class T>
__global__ void k_dot_free(int64_t N, const uint8_t *__restrict__ flag, const uint8_t *__restrict__ own,
                           const vec4<T> *__restrict__ a, const vec4<T> *__restrict__ b, double *out) {
    double s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (flag[i] != 1 || !own[i]) continue;
        vec4<T> x = a[i], y = b[i];
        s += (double)(x.x * y.x + x.y * y.y + x.z * y.z);
    }
    block_add(s, out);
}

// vt = v + alpha x on free nodes, v elsewhere
template <class T>
__global__ void k_axpy_free(int64_t N, const uint8_t *__restrict__ flag, T alpha, const vec4<T> *__restrict__ v,
                            const vec4<T> *__restrict__ x, vec4<T> *__restrict__ vt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        vec4<T> a = v[i];
        if (flag[i] == 1) {
            vec4<T> b = x[i];
            a.x += alpha * b.x; a.y += alpha * b.y; a.z += alpha * b.z;
        }
        vt[i] = a;
    }
}

template <class T>
__global__ void k_canon_to_tile(int64_t n, const int *__restrict__ list, const T *__restrict__ src,
                                vec4<T> *__restrict__ dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[list[i]] = mk4<T>(src[3 * i], src[3 * i + 1], src[3 * i + 2], T(0));
}
template <class T>
__global__ void k_tile_to_canon(int64_t n, const int *__restrict__ list, const vec4<T> *__restrict__ src,
                                T *__restrict__ dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        vec4<T> v = src[list[i]];
        dst[3 * i] = v.x; dst[3 * i + 1] = v.y; dst[3 * i + 2] = v.z;
    }
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }
inline unsigned vgrid(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

// =============================================================================================
// host side
// =============================================================================================
template <class T>
mpl_status canon_to_tile(mpl_ctx ctx, const void *src, void *dst_tile) {
    const int64_t n = ctx->n_nodes_active, NT = (int64_t)ctx->T * 64;
    cudaStream_t st = ctx->stream;
    MPL_CHECK(ensure(ctx, ctx->io_stage, (size_t)(n * 3 + 4) * sizeof(T)));
    MPL_CUDA(cudaMemcpyAsync(ctx->io_stage.p, src, n * 3 * sizeof(T), cudaMemcpyDefault, st));
    MPL_CUDA(cudaMemsetAsync(dst_tile, 0, NT * sizeof(vec4<T>), st));
    if (n) k_canon_to_tile<T><<<nblk(n, 256), 256, 0, st>>>(n, (const int *)ctx->n_list.p, (const T *)ctx->io_stage.p,
                                                          (vec4<T> *)dst_tile); ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

template <class T>
mpl_status tile_to_canon(mpl_ctx ctx, const void *src_tile, void *dst) {
    const int64_t n = ctx->n_nodes_active;
    cudaStream_t st = ctx->stream;
    MPL_CHECK(ensure(ctx, ctx->io_stage, (size_t)(n * 3 + 4) * sizeof(T)));
    if (n) k_tile_to_canon<T><<<nblk(n, 256), 256, 0, st>>>(n, (const int *)ctx->n_list.p, (const vec4<T> *)src_tile,
                                                          (T *)ctx->io_stage.p); ctx->launches++;
    MPL_CUDA(cudaMemcpyAsync(dst, ctx->io_stage.p, n * 3 * sizeof(T), cudaMemcpyDefault, st));
    MPL_CHECK(d2h_sync(ctx, st));
    return MPL_OK;
}

// Launch the linearisation kernel at v_tile; writes g (n_g), diag (n_diag), K; returns Phi.
template <class T>
mpl_status linearize_impl(mpl_ctx ctx, const void *v_tile, int mode, double *phi) {
    cudaStream_t st = ctx->stream;
#ifdef MPL_DEBUG
    MPL_CHECK(debug_check_tiles(ctx, "linearize"));
#endif
    const int T_ = ctx->T;
    const int64_t NT = (int64_t)T_ * 64;
    DevScalars *sc = (DevScalars *)ctx->scalars.p;
    MPL_CUDA(cudaMemsetAsync(sc->energy, 0, sizeof(sc->energy) + sizeof(double), st));  // + inv_any
    if (mode != LIN_ENERGY) MPL_CUDA(cudaMemsetAsync(ctx->n_g.p, 0, NT * sizeof(vec4<T>), st));
    if (mode == LIN_FULL) MPL_CUDA(cudaMemsetAsync(ctx->n_diag.p, 0, NT * sizeof(vec4<T>), st));
    if (T_) {
#define LIN_ARGS                                                                                                  \
    ctx->grid, ctx->mats, ctx->dt, (const int *)ctx->t_nplus.p, (const int *)ctx->t_cstart.p,                     \
        (const uint8_t *)ctx->c_local.p, (const int *)ctx->t_hascells.p, (const vec4<T> *)v_tile,                  \
        (const vec4<T> *)ctx->n_vhat.p, (const T *)owned_mass(ctx), (const T *)ctx->q_slot.p, (T *)ctx->K.p,       \
        (const int *)(kc ? ctx->t_kstart2.p : ctx->t_kstart.p), (const int *)ctx->t_ncell.p, (vec4<T> *)ctx->n_g.p, \
        (vec4<T> *)ctx->n_diag.p,                                                                                 \
        ctx->mats.plastic ? (T *)ctx->q_Sp.p : (T *)nullptr, sc, hvp_kz_layout(ctx->precision), kc
        // 64 threads per tile: one per cell (a tile has <= 64); 128 left half the CTA idle in the
        // cell phase (ncu at cfg4: barrier stalls 34 %, 16 warps / SM by registers)
        const char *lte = getenv("MPL_LIN_THREADS");
        const int lt = lte ? atoi(lte) : 64;
        const char *lge = getenv("MPL_LIN_GEN_MINB");
        const int lin_gen_minb = lge ? atoi(lge) : 12;  // 12 CTAs per SM (NH / water / VM linearisations -7 %)
        bool honly = !ctx->mats.plastic;
        for (int k = 0; k < ctx->mats.nmat; k++) honly = honly && ctx->mats.kind[k] == 0;
        // compressed tangent (MPL_KC, default on): fp32 k_hvp_wz, StVK-Hencky elastic only, exact Hessian,
        // one occupied material slot per cell
        const char *kce = getenv("MPL_KC");
        const int kc = (mode == LIN_FULL && sizeof(T) == 4 && honly && (!ctx->psd_now || ctx->nonid_base_cells == 0) &&
                        hvp_variant() == 0 && ctx->multi_slot_cells == 0 && !(kce && kce[0] == '0')) ? 1 : 0;
        if (mode == LIN_FULL) ctx->kc_now = kc;
        if (mode == LIN_FULL && ctx->psd_now) {  // per-cell PSD projection of K
            // launch bounds (128, 1): the register-resident Jacobi (126 live reals) needs the registers
            if (honly && kc) k_linearize<T, LIN_FULL, true, 1, true, true><<<T_, 64, 0, st>>>(LIN_ARGS);
            else if (honly) k_linearize<T, LIN_FULL, true, 1, true><<<T_, 64, 0, st>>>(LIN_ARGS);
            else k_linearize<T, LIN_FULL, false, 1, true><<<T_, 64, 0, st>>>(LIN_ARGS);
        } else if (honly) {
            if (mode == LIN_ENERGY) k_linearize<T, LIN_ENERGY, true><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (mode == LIN_GRAD) k_linearize<T, LIN_GRAD, true><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (lt == 64 && kc) k_linearize<T, LIN_FULL, true, 12, false, true><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (lt == 64) k_linearize<T, LIN_FULL, true, 12><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (kc) k_linearize<T, LIN_FULL, true, 1, false, true><<<T_, lt, 0, st>>>(LIN_ARGS);
            else k_linearize<T, LIN_FULL, true><<<T_, lt, 0, st>>>(LIN_ARGS);
        } else {
            if (mode == LIN_ENERGY) k_linearize<T, LIN_ENERGY><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (mode == LIN_GRAD) k_linearize<T, LIN_GRAD><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (lt == 64 && lin_gen_minb == 12) k_linearize<T, LIN_FULL, false, 12><<<T_, lt, 0, st>>>(LIN_ARGS);
            else if (lt == 64) k_linearize<T, LIN_FULL, false, 8><<<T_, lt, 0, st>>>(LIN_ARGS);
            else k_linearize<T, LIN_FULL><<<T_, lt, 0, st>>>(LIN_ARGS);
        }
        ctx->launches++;
#undef LIN_ARGS
    }
    MPL_CUDA(cudaGetLastError());
    // slab ranks: complete g / diag on the shared node planes, sum Phi over ranks
    if (mode != LIN_ENERGY) MPL_CHECK(halo_sum_nodes<T>(ctx, ctx->n_g.p, mode == LIN_FULL ? ctx->n_diag.p : nullptr));
    MPL_CHECK(allreduce_d(ctx, sc->energy, NSTRIPE + 1));
    if (phi) {
        double e[NSTRIPE + 1];
        MPL_CHECK(d2h(ctx, e, sc->energy, sizeof e, st));
        MPL_CHECK(d2h_sync(ctx, st));
        *phi = e[NSTRIPE] != 0.0 ? __builtin_inf() : host_stripes(e);
    }
    if (mode == LIN_FULL) ctx->linearized = true;
    return MPL_OK;
}

// One HVP on tile-dense vectors: Hu = H u (Hu zeroed here); optional u.Hu accumulation.
template <class T>
mpl_status hvp_tile(mpl_ctx ctx, const void *u_tile, void *Hu_tile, double *uHu_accum) {
    MPL_CUDA(cudaMemsetAsync(Hu_tile, 0, (size_t)ctx->T * 64 * sizeof(vec4<T>), ctx->stream));
    MPL_CHECK(launch_hvp<T>(ctx, u_tile, Hu_tile, uHu_accum, nullptr, 0, 0.0));
    return halo_sum_nodes<T>(ctx, Hu_tile, nullptr);
}

namespace {
template <class T>
mpl_status energy_at(mpl_ctx ctx, const void *v_tile, double *phi) {
    return linearize_impl<T>(ctx, v_tile, LIN_ENERGY, phi);
}
}  // namespace

constexpr int HVP_SAMPLE = 16;  // every 16th HVP bracketed by events (each pair ~6 us and a broken PDL overlap)

template <class T>
mpl_status newton_impl(mpl_ctx ctx, const mpl_solver_cfg *cfg, mpl_solve_stats *out) {
    cudaStream_t st = ctx->stream;
    const int64_t NT = (int64_t)ctx->T * 64;
    DevScalars *sc = (DevScalars *)ctx->scalars.p;
    mpl_solve_stats S{};
    // Hessian used by this solve: exact (amb-6, negative-curvature stop) or per-cell PSD-projected
    struct PsdGuard {
        mpl_ctx c;
        int old;
        ~PsdGuard() { c->psd_now = old; }
    } psd_guard{ctx, ctx->psd_now};
    ctx->psd_now = cfg->psd_project ? 1 : 0;
    const bool fixed = cfg->fixed_newton_iters > 0;
    const int kmax = fixed ? cfg->fixed_newton_iters : cfg->newton_max;
    const int cg_cap = cfg->cg_max > 0 ? cfg->cg_max : 1;
    int slots_needed = cg_cap + 2;
    if (cfg->fixed_cg_iters)
        for (int k = 0; k < kmax; k++) slots_needed = std::max(slots_needed, cfg->fixed_cg_iters[k] + 2);
    MPL_CHECK(ensure(ctx, ctx->cg_slots, (size_t)slots_needed * sizeof(CGSlot)));
    CGSlot *slots = (CGSlot *)ctx->cg_slots.p;
    const uint8_t *flag = (const uint8_t *)ctx->n_flag.p;
    const uint8_t *own = (const uint8_t *)ctx->n_own.p;
    vec4<T> *v = (vec4<T> *)ctx->n_v.p, *vt = (vec4<T> *)ctx->n_vt.p;
    vec4<T> *g = (vec4<T> *)ctx->n_g.p, *D = (vec4<T> *)ctx->n_diag.p;
    const int64_t NA = ctx->n_nodes_active;
    const int64_t SA = soa_stride(NA);  // SoA stride of x, r, invD (3 SA reals each)
    MPL_CHECK(ensure(ctx, ctx->n_invD, (size_t)3 * SA * sizeof(T) + 64));
    MPL_CHECK(ensure(ctx, ctx->n_x, (size_t)3 * SA * sizeof(T) + 64));
    MPL_CHECK(ensure(ctx, ctx->n_r, (size_t)3 * SA * sizeof(T) + 64));
    T *invD = (T *)ctx->n_invD.p, *x = (T *)ctx->n_x.p, *r = (T *)ctx->n_r.p;
    // p and Hp in one allocation (Hp = p + NT), so one L2 access-policy window can cover both
    // cg1 keeps a second HVP output buffer: the vector kernel of iteration j zeroes w_j while HVP_{j+1}
    // writes the other one, zeroed an iteration earlier (zeroing right before the HVP that writes the same
    // buffer left its dirty lines to be written back during that HVP)
    MPL_CHECK(ensure(ctx, ctx->n_p, (size_t)3 * NT * sizeof(vec4<T>) + 64));
    vec4<T> *p = (vec4<T> *)ctx->n_p.p, *Hp = p + NT;
    const uint8_t *own_w = multi(ctx) ? own : nullptr;  // dot-product owner weights (slab ranks)
    // PCG form (MPL_PCG): "cg1" single-reduction recurrence (one vector kernel and one allreduce per
    // iteration: the default on slab ranks, where an allreduce costs more than the kernel) or "classic"
    // Hestenes-Stiefel with two vector kernels (the default on one GPU: cfg4 PCG 50.7 ms vs 56.1 ms cg1,
    // whose 13-stream vector kernel runs 71 us vs 60 us for the two, and whose HVP writes into a w
    // zeroed one iteration earlier: 100.6 vs 95.2 us; profiles/r02_pcg_forms.json)
    const char *pcge = getenv("MPL_PCG");
    const bool cg1 = pcge ? pcge[0] != 'c' : multi(ctx);
    const char *cge = getenv("MPL_CG1_E");  // nodes per lane per chunk of the cg1 vector kernel (2 or 4)
    const int cg1_e = cge ? atoi(cge) : 2;
    T *pc = nullptr, *sc_ = nullptr;  // cg1: compact p, s
    // slab ranks, cg1, k_hvp_wz: the HVP in two launches (interface tiles, then interior) with the face halo
    // between them (MPL_OVERLAP=0 disables); on the NCCL transport the halo runs on its own stream,
    // concurrently with the interior launch
    const char *ove = getenv("MPL_OVERLAP");
    const bool split = cg1 && multi(ctx) && sizeof(T) == 4 && hvp_variant() == 0 && !(ove && ove[0] == '0');
    const bool overlap = split && comm_is_nccl(ctx);
    if (overlap && !ctx->hstream) {
        MPL_CUDA(cudaStreamCreateWithFlags(&ctx->hstream, cudaStreamNonBlocking));
        MPL_CUDA(cudaEventCreateWithFlags(&ctx->ev_bnd, cudaEventDisableTiming));
        MPL_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
    }
    if (cg1) {
        MPL_CHECK(ensure(ctx, ctx->n_ps, (size_t)6 * SA * sizeof(T) + 64));
        pc = (T *)ctx->n_ps.p;
        sc_ = pc + 3 * SA;
    }
    const char *pme = getenv("MPL_PCG_MAP");
    // warp-interleaved update kernels (fp32 default; the fp64 instances spill, MPL_PCG_MAP=group / warp)
    const bool pcg_warp_map = pme ? pme[0] == 'w' : sizeof(T) == 4;
    const char *pmb = getenv("MPL_PCG_MINB");  // CTAs of 256 per SM requested from ptxas (2: <= 128 registers)
    const int pcg_minb = pmb ? atoi(pmb) : 2;
    // MPL_PCG_Z (fp32 warp-map kernels, default 1): the residual buffer holds z = D^-1 r instead of r
    // (update2 then reads z instead of r and D^-1: 12 B per node less; r = D z for the dot products).
    // cfg4: update2 10.75 -> 9.43 ms, update1 12.15 -> 12.55 ms per step (the divisions), step 54.5 -> 53.7 ms
    const char *pze = getenv("MPL_PCG_Z");
    const bool pcg_z = !cg1 && sizeof(T) == 4 && pcg_warp_map && pcg_minb == 2 && !(pze && pze[0] == '0');
    // MPL_PCG_GRAPH=1 (one GPU, fp32 compressed tangent, classic z-form PCG): two PCG iterations (HVP,
    // update1, update2 each, with their programmatic-launch edges) captured once per step into a CUDA graph
    // and replayed; the kernels read the iteration index and threshold from device memory, update2
    // advancing it (no per-iteration launch arguments), and the convergence test stays on the device.
    // Not the default: the HVP sampling events of the bench need the stream path.
    const char *pge = getenv("MPL_PCG_GRAPH");
    const bool pcg_graph = pge && pge[0] == '1' && pcg_z && !multi(ctx) && ctx->kc_now && hvp_variant() == 0;
    cudaGraphExec_t pcg_gexec = nullptr;
    struct GraphGuard {
        cudaGraphExec_t *g;
        ~GraphGuard() {
            if (*g) cudaGraphExecDestroy(*g);
        }
    } pcg_gguard{&pcg_gexec};
    const unsigned VG = vgrid(NT);
    const unsigned VA = vgrid(NA);
    const unsigned VA1 = nblk(NA > 0 ? NA : 1, 256);
    int nsm_ = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm_, cudaDevAttrMultiProcessorCount, dev);
    }
    // persistent update kernels: MPL_PCG_CPS CTAs per SM; the fp32 warp-map kernels default to the 2 that
    // are resident (one wave; cfg4 vector kernels 22.1 -> 21.3 ms per step against 8 = four waves)
    const char *cpse = getenv("MPL_PCG_CPS");
    const int cps = cpse ? atoi(cpse) : (sizeof(T) == 4 && pcg_warp_map && pcg_minb == 2) ? 2 : 8;
    const unsigned VAP = std::min<unsigned>(VA1, (unsigned)nsm_ * cps);
    const int *list = (const int *)ctx->n_list.p;
    // L2 persisting access-policy window for the Newton solve over p (MPL_L2WIN=p, default: the HVP's
    // gathered input, read by update2), Hp (=h: the HVP's atomics target) or both at half hit ratio
    // (=ph); without it the 390 MB tangent and the vector streams evict them between kernels.  Measured
    // at cfg4 (step ms / in-step HVP us): none 66.1 / 100.3, p 64.6 / 95.7, h 64.5 / 96.4, ph 65.2 /
    // 96.9; both at full hit ratio (74 MB of the 126 MB L2) 71.3 / 103.5.  MPL_L2WIN=0 disables;
    // After the solve the persisting lines are reset (MPL_L2RESET=0 keeps them); the persisting limit is
    // set once, not released: cudaDeviceSetLimit synchronises the device, and calling it per solve
    // serialised the pipelined host copies (e2e 102 -> 119 ms / step at cfg4).
    const char *l2w = getenv("MPL_L2WIN");
    const int l2mode = !l2w ? 2 : l2w[0] == '0' ? 0 : l2w[0] == 'h' ? 1 : (l2w[0] == 'p' && l2w[1] == 'h') ? 3 : 2;
    const char *l2r = getenv("MPL_L2RESET");
    const bool l2reset = !(l2r && l2r[0] == '0');
    bool l2on = l2mode != 0;
    if (l2on) {
        int dev = 0, maxp = 0, maxw = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t vb = (size_t)NT * sizeof(vec4<T>);
        const size_t want = l2mode == 3 ? 2 * vb : vb;
        const size_t win = std::min(want, (size_t)maxw);
        const size_t lim = std::min(vb, (size_t)maxp);
        // only when the window is fully persisting: a partial hit ratio (cfg5: p = 232 MB) halved the
        // HVP's speed in the solve and after it
        if (win > lim || lim == 0) l2on = false;
        static size_t limit_set = 0;  // cudaDeviceSetLimit synchronises the device: only on a change
        if (l2on && limit_set != lim) {
            MPL_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim));
            limit_set = lim;
        }
        if (l2on) {
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.base_ptr = (void *)(l2mode == 1 ? Hp : p);
            a.accessPolicyWindow.num_bytes = win;
            a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)lim / (double)win);
            a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            MPL_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));
        }
    }
    // the window is cleared (and the persisting lines reset) however the solve returns
    struct L2WindowGuard {
        cudaStream_t st;
        bool on, reset;
        ~L2WindowGuard() {
            if (!on) return;
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.num_bytes = 0;
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
            if (reset) cudaCtxResetPersistingL2Cache();
        }
    } l2guard{st, l2on, l2reset};
    cudaEvent_t e0, e1, h0, h1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> hev;
    std::vector<std::pair<int, int>> sampled;  // (event pair, PCG iteration) of timed HVP launches
    int nl = 0;                                // HVP launches (incl. ones skipped after convergence)
    double hvp_sample_ms = 0.0;
    int hvp_sample_n = 0;
    // per-HVP device timing (stats.hvp_ms): CUDA events around every HVP_SAMPLE-th HVP launch (the
    // events cost ~4 us each inside the PCG loop); MPL_HVP_EVENTS=0 drops them
    const char *hve = getenv("MPL_HVP_EVENTS");
    const bool hvp_events = !(hve && hve[0] == '0');
    // MPL_VEC_EVENTS=1: also time the PCG vector kernels (stats.ms_phase[1])
    const char *vee = getenv("MPL_VEC_EVENTS");
    const bool vec_events = vee && (vee[0] == '1' || vee[0] == '2') && !cg1;  // classic PCG only
    std::vector<std::array<cudaEvent_t, 3>> vev;  // before update1, between, after update2
    double t_lin = 0, t_pcg = 0, t_ls = 0;
    auto elapsed = [&](cudaEvent_t a, cudaEvent_t b) {
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return (double)ms;
    };
    std::vector<CGSlot> hslots;
    double phi0 = 0;
    double phi_v = 0;       // Phi at the current v when known (the linearisation at v, or the accepted trial)
    bool phi_known = false;
    for (int k = 0; k < kmax; k++) {
        // ---- linearise at v^k -------------------------------------------------------------
        cudaEventRecord(e0, st);
        MPL_CHECK(linearize_impl<T>(ctx, v, LIN_FULL, nullptr));
        MPL_CUDA(cudaMemsetAsync(slots, 0, slots_needed * sizeof(CGSlot), st));
        MPL_CUDA(cudaMemsetAsync(&sc->neg_curv, 0, sizeof(int), st));
        MPL_CUDA(cudaMemsetAsync(&sc->cg_done_iter, 0xff, sizeof(int), st));
        MPL_CUDA(cudaMemsetAsync(p, 0, NT * sizeof(vec4<T>), st));
        k_pcg_init<T><<<vgrid(SA), 256, 0, st>>>(NA, SA, list, flag, own_w, g, D, invD, r, p, x, slots, pcg_z);
        ctx->launches++;
        MPL_CHECK(allreduce_d(ctx, slots[0].rz, 3 * NSTRIPE));
        MPL_CUDA(cudaMemsetAsync(Hp, 0, NT * sizeof(vec4<T>), st));
        if (cg1) {
            MPL_CUDA(cudaMemsetAsync(pc, 0, (size_t)6 * SA * sizeof(T), st));  // p_{-1} = s_{-1} = 0
            MPL_CUDA(cudaMemsetAsync(Hp + NT, 0, NT * sizeof(vec4<T>), st));  // the second w buffer
        }
        cudaEventRecord(e1, st);
        CGSlot s0;
        double e[NSTRIPE + 1];
        MPL_CHECK(d2h(ctx, &s0, slots, sizeof s0, st));
        MPL_CHECK(d2h(ctx, e, sc->energy, sizeof e, st));
        MPL_CHECK(d2h_sync(ctx, st));
        t_lin += elapsed(e0, e1);
        phi0 = e[NSTRIPE] != 0.0 ? __builtin_inf() : host_stripes(e);
        phi_v = phi0;
        phi_known = true;
        const double rr0 = host_stripes(s0.rr);
        const double gn = sqrt(rr0);
        if (k == 0) S.grad_norm0 = gn;
        S.grad_norm = gn;
        if (k < MPL_MAX_NEWTON_LOG) S.grad_norms[k] = gn;
        if (!fixed && gn <= cfg->newton_rtol * S.grad_norm0) {
            S.converged = 1;
            break;
        }
        // ---- PCG on H x = -g -----------------------------------------------------------------
        const int itmax = cfg->fixed_cg_iters ? cfg->fixed_cg_iters[k] : cg_cap;
        const double thr = cfg->fixed_cg_iters ? -1.0 : cfg->cg_rtol * cfg->cg_rtol * rr0;
        int launched = 0, its = 0;
        cudaEventRecord(e0, st);
        if (pcg_graph && rr0 > 0.0 && itmax > 0) {
            k_set_cg<<<1, 1, 0, st>>>(sc, thr);
            ctx->launches++;
            if (!pcg_gexec) {  // capture two iterations (even: reads cg_j[0], writes cg_j[1]; odd: back)
                cudaGraph_t gr = nullptr;
                MPL_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
                mpl_status cs_ = MPL_OK;
                for (int par = 0; par < 2 && cs_ == MPL_OK; par++) {
                    const int *jin = &sc->cg_j[par];
                    int *jo = &sc->cg_j[par ^ 1];
                    cs_ = launch_hvp<T>(ctx, p, Hp, nullptr, slots, 0, thr, nullptr, 0, jin);
                    if (cs_ == MPL_OK &&
                        launch_pdl(k_pcg_update1w<T, PCG_E, 2, true>, VAP, 256, 0, st, NA, SA, list, 0, thr, invD, p,
                                   Hp, x, r, own_w, slots, sc, jin) != cudaSuccess)
                        cs_ = MPL_ERR_CUDA;
                    if (cs_ == MPL_OK &&
                        launch_pdl(k_pcg_update2w<T, PCG_E, 2, true>, VAP, 256, 0, st, NA, SA, list, 0, thr, invD, r,
                                   p, x, slots, sc, jin, jo) != cudaSuccess)
                        cs_ = MPL_ERR_CUDA;
                }
                const cudaError_t ce = cudaStreamEndCapture(st, &gr);
                MPL_CHECK(cs_);
                MPL_CUDA(ce);
                const cudaError_t ie = cudaGraphInstantiate(&pcg_gexec, gr, 0);
                cudaGraphDestroy(gr);
                MPL_CUDA(ie);
                ctx->launches -= 2;  // launch_hvp counted the captured HVPs
            }
        }
        if (rr0 > 0.0 && itmax > 0) {
            int chunk = 4;
            bool done = false;
            while (!done && launched < itmax) {
                int n = std::min(chunk, itmax - launched);
                if (pcg_graph) {  // pairs of iterations by graph replay; an odd last iteration on the stream path
                    n = std::min((chunk + 1) & ~1, itmax - launched);
                    for (int q = 0; q < n / 2; q++) MPL_CUDA(cudaGraphLaunch(pcg_gexec, st));
                    ctx->launches += 6 * (n / 2);
                    nl += 2 * (n / 2);
                }
                for (int jj = launched + (pcg_graph ? 2 * (n / 2) : 0); jj < launched + n; jj++) {
                    if ((int)hev.size() <= nl) {
                        cudaEvent_t a, b;
                        cudaEventCreate(&a);
                        cudaEventCreate(&b);
                        hev.push_back({a, b});
                        if (vec_events) {
                            std::array<cudaEvent_t, 3> ev;
                            for (auto &x : ev) cudaEventCreate(&x);
                            vev.push_back(ev);
                        }
                    }
                    const bool timed = hvp_events && (jj % HVP_SAMPLE == 0);
                    if (cg1) {
                        // iteration jj: [HVP_0 once] -> vector kernel jj -> HVP_{jj+1} (+ halo, one allreduce)
                        auto wbuf = [&](int i) { return Hp + (int64_t)(i & 1) * NT; };  // w_i
                        if (jj == 0) {
                            if (timed) cudaEventRecord(hev[nl].first, st);
                            MPL_CHECK(launch_hvp<T>(ctx, p, wbuf(0), slots[0].pHp, slots, 0, thr));
                            if (multi(ctx)) {
                                MPL_CHECK(halo_sum_nodes<T>(ctx, wbuf(0), nullptr));
                                MPL_CHECK(allreduce_d(ctx, slots[0].pHp, NSTRIPE));
                            }
                            if (timed) {
                                cudaEventRecord(hev[nl].second, st);
                                sampled.push_back({nl, 0});
                            }
                            nl++;
                            if ((int)hev.size() <= nl) {
                                cudaEvent_t a, b;
                                cudaEventCreate(&a);
                                cudaEventCreate(&b);
                                hev.push_back({a, b});
                            }
                        }
                        if (cg1_e == 4)
                            MPL_CUDA(launch_pdl(k_pcg_cg1<T, 4>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p, wbuf(jj),
                                                x, r, pc, sc_, own_w, slots, sc));
                        else
                            MPL_CUDA(launch_pdl(k_pcg_cg1<T, 2>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p, wbuf(jj),
                                                x, r, pc, sc_, own_w, slots, sc));
                        ctx->launches++;
                        const bool timed1 = hvp_events && ((jj + 1) % HVP_SAMPLE == 0);
                        if (timed1) cudaEventRecord(hev[nl].first, st);
                        // on slab ranks slot jj+1 is not reduced yet: skip on the previous (reduced) residual
                        const int cgj1 = multi(ctx) ? jj : jj + 1;
                        if (split) {
                            // interface tiles first; their face halo runs (NCCL: on the halo stream, concurrent
                            // with the interior tiles) while the interior tiles, which touch no shared node, run
                            MPL_CHECK(launch_hvp<T>(ctx, p, wbuf(jj + 1), slots[jj + 1].pHp, slots, cgj1, thr,
                                                    (const int *)ctx->t_bnd.p, ctx->n_bnd));
                            if (overlap) {
                                MPL_CUDA(cudaEventRecord(ctx->ev_bnd, st));
                                MPL_CUDA(cudaStreamWaitEvent(ctx->hstream, ctx->ev_bnd, 0));
                                ctx->stream = ctx->hstream;
                                const mpl_status hs = halo_sum_nodes<T>(ctx, wbuf(jj + 1), nullptr);
                                ctx->stream = st;
                                MPL_CHECK(hs);
                                MPL_CUDA(cudaEventRecord(ctx->ev_halo, ctx->hstream));
                            } else {
                                MPL_CHECK(halo_sum_nodes<T>(ctx, wbuf(jj + 1), nullptr));
                            }
                            MPL_CHECK(launch_hvp<T>(ctx, p, wbuf(jj + 1), slots[jj + 1].pHp, slots, cgj1, thr,
                                                    (const int *)ctx->t_int.p, ctx->n_int));
                            if (overlap) MPL_CUDA(cudaStreamWaitEvent(st, ctx->ev_halo, 0));
                            MPL_CHECK(allreduce_d(ctx, slots[jj + 1].rz, 3 * NSTRIPE));  // gamma, r.r, delta
                        } else {
                            MPL_CHECK(launch_hvp<T>(ctx, p, wbuf(jj + 1), slots[jj + 1].pHp, slots, cgj1, thr));
                            if (multi(ctx)) {
                                MPL_CHECK(halo_sum_nodes<T>(ctx, wbuf(jj + 1), nullptr));
                                MPL_CHECK(allreduce_d(ctx, slots[jj + 1].rz, 3 * NSTRIPE));  // gamma, r.r, delta
                            }
                        }
                        if (timed1) {
                            cudaEventRecord(hev[nl].second, st);
                            sampled.push_back({nl, jj + 1});
                        }
                        nl++;
                        continue;
                    }
                    if (timed) cudaEventRecord(hev[nl].first, st);
                    // the HVP is skipped on device once converged (its output is then unused)
                    MPL_CHECK(launch_hvp<T>(ctx, p, Hp, slots[jj].pHp, slots, jj, thr));
                    if (multi(ctx)) {  // complete Hp on the shared planes; global p.Hp (timed with the HVP)
                        MPL_CHECK(halo_sum_nodes<T>(ctx, Hp, nullptr));
                        MPL_CHECK(allreduce_d(ctx, slots[jj].pHp, NSTRIPE));
                    }
                    if (timed) cudaEventRecord(hev[nl].second, st);
                    if (timed) sampled.push_back({nl, jj});
                    nl++;
                    if (vec_events) cudaEventRecord(vev[nl - 1][0], st);
                    if (pcg_z)
                        MPL_CUDA(launch_pdl(k_pcg_update1w<T, PCG_E, 2, true>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD,
                                            p, Hp, x, r, own_w, slots, sc, (const int *)nullptr));
                    else if (pcg_warp_map && pcg_minb == 3)
                        MPL_CUDA(launch_pdl(k_pcg_update1w<T, PCG_E, 3>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p,
                                            Hp, x, r, own_w, slots, sc, (const int *)nullptr));
                    else if (pcg_warp_map && pcg_minb == 4)
                        MPL_CUDA(launch_pdl(k_pcg_update1w<T, PCG_E, 4>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p,
                                            Hp, x, r, own_w, slots, sc, (const int *)nullptr));
                    else if (pcg_warp_map)
                        MPL_CUDA(launch_pdl(k_pcg_update1w<T>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p, Hp, x,
                                            r, own_w, slots, sc, (const int *)nullptr));
                    else
                        MPL_CUDA(launch_pdl(k_pcg_update1<T, PCG_U>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, p,
                                            Hp, x, r, own_w, slots, sc));
                    ctx->launches++;
                    MPL_CHECK(allreduce_d(ctx, slots[jj + 1].rz, 2 * NSTRIPE));  // rz, rr of iteration jj+1
                    if (vec_events) cudaEventRecord(vev[nl - 1][1], st);
                    if (pcg_z)
                        MPL_CUDA(launch_pdl(k_pcg_update2w<T, PCG_E, 2, true>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD,
                                            r, p, x, slots, sc, (const int *)nullptr, (int *)nullptr));
                    else if (pcg_warp_map && pcg_minb == 3)
                        MPL_CUDA(launch_pdl(k_pcg_update2w<T, PCG_E, 3>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, r,
                                            p, x, slots, sc, (const int *)nullptr, (int *)nullptr));
                    else if (pcg_warp_map && pcg_minb == 4)
                        MPL_CUDA(launch_pdl(k_pcg_update2w<T, PCG_E, 4>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, r,
                                            p, x, slots, sc, (const int *)nullptr, (int *)nullptr));
                    else if (pcg_warp_map)
                        MPL_CUDA(launch_pdl(k_pcg_update2w<T>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, r, p, x,
                                            slots, sc, (const int *)nullptr, (int *)nullptr));
                    else
                        MPL_CUDA(launch_pdl(k_pcg_update2<T, PCG_U>, VAP, 256, 0, st, NA, SA, list, jj, thr, invD, r,
                                            p, x, slots, sc));
                    ctx->launches++;
                    if (vec_events) cudaEventRecord(vev[nl - 1][2], st);
                }
                launched += n;
                MPL_CUDA(cudaGetLastError());
                CGSlot sl;
                int neg = 0;
                MPL_CHECK(d2h(ctx, &sl, slots + launched, sizeof sl, st));
                MPL_CHECK(d2h(ctx, &neg, &sc->neg_curv, sizeof neg, st));
                MPL_CHECK(d2h_sync(ctx, st));
                const double rr_now = host_stripes(sl.rr);
                if (neg || rr_now <= thr) done = true;
                // next chunk: the iterations the residual's average decay so far predicts to the
                // threshold (+2), between 4 and 64 (every launch past convergence exits at once on the
                // device but still costs its launch; every chunk costs a host round trip)
                int next = std::min(chunk * 2, 64);
                if (!done && thr > 0.0 && rr_now > 0.0 && rr_now < rr0) {
                    const double rate = std::log(rr_now / rr0) / (double)launched;  // < 0 per iteration
                    const double need = std::log(thr / rr_now) / rate;
                    if (need > 0.0 && need < 1e6) next = std::max(4, std::min(64, (int)std::ceil(need) + 2));
                }
                chunk = next;
            }
            hslots.resize(launched + 1);
            int neg = 0, doneit = -1;
            MPL_CHECK(d2h(ctx, hslots.data(), slots, (launched + 1) * sizeof(CGSlot), st));
            MPL_CHECK(d2h(ctx, &neg, &sc->neg_curv, sizeof neg, st));
            MPL_CHECK(d2h(ctx, &doneit, &sc->cg_done_iter, sizeof doneit, st));
            MPL_CHECK(d2h_sync(ctx, st));
            its = launched;
            if (neg) {
                its = doneit;
                S.neg_curvature++;
            } else {
                for (int s = 1; s <= launched; s++)
                    if (host_stripes(hslots[s].rr) <= thr) { its = s; break; }
            }
        }
        cudaEventRecord(e1, st);
        MPL_CUDA(cudaEventSynchronize(e1));
        t_pcg += elapsed(e0, e1);
        // HVPs launched past convergence exit on the device at once: only iterations jj < its count
        for (const auto &sp : sampled)
            if (sp.second < its) {
                hvp_sample_ms += elapsed(hev[sp.first].first, hev[sp.first].second);
                hvp_sample_n++;
            }
        sampled.clear();
        S.n_hvp += its;
        if (k < MPL_MAX_NEWTON_LOG) S.cg_iters[k] = its;
        S.cg_iters_total += its;
        // ---- Armijo backtracking line search ------------------------------------------------
        cudaEventRecord(e0, st);
        MPL_CUDA(cudaMemsetAsync(sc->gp, 0, sizeof(sc->gp), st));
        k_dot_gx<T><<<VA, 256, 0, st>>>(NA, SA, list, flag, own, g, x, sc->gp); ctx->launches++;
        MPL_CHECK(allreduce_d(ctx, sc->gp, NSTRIPE));
        double gps[NSTRIPE];
        MPL_CHECK(d2h(ctx, gps, sc->gp, sizeof gps, st));
        MPL_CHECK(d2h_sync(ctx, st));
        const double gp = host_stripes(gps);
        double alpha = 1.0;
        int h = 0;
        double phi_acc = 0;
        bool phi_acc_known = false;
        if (cfg->fixed_ls_halvings) {
            for (h = 0; h < cfg->fixed_ls_halvings[k]; h++) alpha *= 0.5;
            MPL_CUDA(cudaMemcpyAsync(vt, v, NT * sizeof(vec4<T>), cudaMemcpyDeviceToDevice, st));
            k_axpy_compact<T><<<VA, 256, 0, st>>>(NA, SA, list, flag, T(alpha), v, x, vt); ctx->launches++;
        } else {
            for (;;) {
                MPL_CUDA(cudaMemcpyAsync(vt, v, NT * sizeof(vec4<T>), cudaMemcpyDeviceToDevice, st));
            k_axpy_compact<T><<<VA, 256, 0, st>>>(NA, SA, list, flag, T(alpha), v, x, vt); ctx->launches++;
                double phi = 0;
                MPL_CHECK(energy_at<T>(ctx, vt, &phi));
                if (std::isinf(phi)) S.n_inverted_trials++;
                phi_acc = phi;
                phi_acc_known = true;
                if (phi <= phi0 + cfg->armijo_c * alpha * gp + cfg->ls_slack * fabs(phi0)) break;
                if (h >= cfg->ls_max) break;
                alpha *= 0.5;
                h++;
            }
        }
        cudaEventRecord(e1, st);
        MPL_CUDA(cudaEventSynchronize(e1));
        t_ls += elapsed(e0, e1);
        if (k < MPL_MAX_NEWTON_LOG) S.ls_iters[k] = h;
        if (k < MPL_MAX_NEWTON_LOG) S.alphas[k] = alpha;
        S.ls_halvings += h;
        std::swap(v, vt);
        std::swap(ctx->n_v, ctx->n_vt);
        phi_v = phi_acc;
        phi_known = phi_acc_known;
        S.newton_iters = k + 1;
    }
    if (!fixed && S.newton_iters == kmax && !S.converged) {
        MPL_CHECK(linearize_impl<T>(ctx, v, LIN_GRAD, nullptr));
        MPL_CUDA(cudaMemsetAsync(sc->gnorm2, 0, sizeof(sc->gnorm2), st));
        k_dot_free<T><<<VG, 256, 0, st>>>(NT, flag, own, g, g, sc->gnorm2); ctx->launches++;
        MPL_CHECK(allreduce_d(ctx, sc->gnorm2, NSTRIPE));
        double g2[NSTRIPE];
        MPL_CHECK(d2h(ctx, g2, sc->gnorm2, sizeof g2, st));
        MPL_CHECK(d2h_sync(ctx, st));
        S.grad_norm = sqrt(host_stripes(g2));
        if (kmax < MPL_MAX_NEWTON_LOG) S.grad_norms[kmax] = S.grad_norm;
        if (S.grad_norm <= cfg->newton_rtol * S.grad_norm0) S.converged = 1;
    }
    // Phi at the returned v: already known from its linearisation or from the accepted line-search trial
    // (one energy pass per step less); computed only after replayed (fixed) line searches
    if (phi_known) S.energy = phi_v;
    else MPL_CHECK(energy_at<T>(ctx, v, &S.energy));
    double hsum = 0;
    if (hvp_events && hvp_sample_n > 0)  // mean of the timed executed HVPs x executed HVPs
        hsum = hvp_sample_ms / hvp_sample_n * S.n_hvp;
    double vsum = 0, v2sum = 0;
    if (vec_events)
        for (int i = 0; i < nl; i++) {
            vsum += elapsed(vev[i][0], vev[i][2]);
            v2sum += elapsed(vev[i][1], vev[i][2]);
        }
    for (auto &ev : vev)
        for (auto &x : ev) cudaEventDestroy(x);
    S.ms_phase[1] = vsum;
    S.ms_phase[2] = v2sum;  // update2 share of ms_phase[1]
    for (auto &pr : hev) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    S.hvp_ms = hsum;
    S.ms_phase[3] = t_lin;
    S.ms_phase[4] = t_pcg;
    S.ms_phase[5] = t_ls;
    ctx->linearized = false;  // K was built at an earlier iterate
    ctx->solved = true;
    S.tangent_format = ctx->kc_now;
    if (out) *out = S;
    (void)h0;
    (void)h1;
    return MPL_OK;
}

// Explicit step velocities (Alg. 3 "Explicit" branch): force into n_g, v^{n+1} into n_v.
template <class T>
mpl_status explicit_impl(mpl_ctx ctx) {
    cudaStream_t st = ctx->stream;
    const int64_t NT = (int64_t)ctx->T * 64, NA = ctx->n_nodes_active;
    MPL_CUDA(cudaMemsetAsync(ctx->n_g.p, 0, NT * sizeof(vec4<T>), st));
    if (ctx->T) {
        k_explicit_force<T><<<ctx->T, 128, 0, st>>>(ctx->grid, ctx->mats.nmat, (const int *)ctx->t_nplus.p,
                                                    (const int *)ctx->t_cstart.p, (const uint8_t *)ctx->c_local.p,
                                                    (const int *)ctx->t_hascells.p, (const T *)ctx->q_slot.p,
                                                    (vec4<T> *)ctx->n_g.p);
        ctx->launches++;
    }
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(halo_sum_nodes<T>(ctx, ctx->n_g.p, nullptr));  // slab ranks: complete f on the shared planes
    if (NA) {
        k_explicit_update<T><<<nblk(NA, 256), 256, 0, st>>>(NA, (const int *)ctx->n_list.p,
                                                            (const uint8_t *)ctx->n_flag.p,
                                                            (const vec4<T> *)ctx->n_vhat.p, (const T *)ctx->n_mass.p,
                                                            (const vec4<T> *)ctx->n_g.p, T(ctx->dt),
                                                            (vec4<T> *)ctx->n_v.p);
        ctx->launches++;
    }
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(d2h_sync(ctx, st));
    ctx->solved = true;
    return MPL_OK;
}

template mpl_status explicit_impl<float>(mpl_ctx);
template mpl_status explicit_impl<double>(mpl_ctx);
template mpl_status canon_to_tile<float>(mpl_ctx, const void *, void *);
template mpl_status canon_to_tile<double>(mpl_ctx, const void *, void *);
template mpl_status tile_to_canon<float>(mpl_ctx, const void *, void *);
template mpl_status tile_to_canon<double>(mpl_ctx, const void *, void *);
template mpl_status linearize_impl<float>(mpl_ctx, const void *, int, double *);
template mpl_status linearize_impl<double>(mpl_ctx, const void *, int, double *);
template mpl_status hvp_tile<float>(mpl_ctx, const void *, void *, double *);
template mpl_status hvp_tile<double>(mpl_ctx, const void *, void *, double *);
template mpl_status newton_impl<float>(mpl_ctx, const mpl_solver_cfg *, mpl_solve_stats *);
template mpl_status newton_impl<double>(mpl_ctx, const mpl_solver_cfg *, mpl_solve_stats *);
