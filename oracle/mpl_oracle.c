/*
 * mpl_oracle.c — CPU fp64 ORACLE for the MPM Lite solve-time hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code, header, table or constant with the CUDA path (paper_2602_07853_b200/csrc)
 * and never reads anything the CUDA path produced.
 *
 * Plain, slow, obviously-correct dense loops in double precision, compiled with
 * -O2 -ffp-contract=off (no fast-math).  Every function cites the passage of
 * /root/reference/PAPER.md ("P:n", section / equation / algorithm) it follows; where
 * the paper is silent the reading is named (amb-#).
 *
 * Grid model: N0 x N1 x N2 cells of size dx, origin o.
 *   node  (i,j,k) at o + dx (i,j,k),            0 <= i <= N0 ...
 *   centre(i,j,k) at o + dx (i+1/2, j+1/2, k+1/2), 0 <= i <  N0 ...
 * All arrays are DENSE over the grid (cells x-major, nodes x-major); a "window"
 * of a large scene is expressed by a smaller grid with a shifted origin.
 * Corner / stencil offsets o in {0,1}^3 are enumerated x-major: o = 4 ox + 2 oy + oz.
 *
 * Threads (OpenMP, optional): the sums over cells that scatter into nodes (gradient, HVP,
 * Jacobi diagonal, explicit force) visit the cells colour by colour, colour = (ci, cj, ck) mod 2,
 * so two cells of one colour never share a node and a colour's cells can run concurrently; the
 * energy and the dot products add fixed per-slice partial sums in a fixed order.  Every result is
 * therefore the same bit for bit at any thread count (OMP_NUM_THREADS); without -fopenmp the
 * pragmas are ignored and the same loops run serially.  Only the order of the terms of each sum
 * differs from a plain x-major loop; the terms are the ones the cited definitions state.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXMAT 8

typedef struct {
    int32_t n[3];
    double dx;
    double origin[3];
} orc_grid;

typedef struct {
    double E, nu, rho;
    int32_t kind; /* 0 = StVK-Hencky, 1 = split Neo-Hookean (App. C),
                     2 = J-based water (kappa = E, Table 2 caption P:536)       */
    double yield_stress; /* von Mises sigma_y (kind 0 only; 0 = elastic): fixed-point plasticity
                            inside Newton ("von Mises", Table 2 "VM: sigma_y") */
} orc_material;

typedef struct {
    double lo[3], hi[3], vel[3];
} orc_box;

/* Solver-time problem: everything Integrate (Alg. 3) reads. */
typedef struct {
    orc_grid g;
    int32_t nmat;
    orc_material mats[ORC_MAXMAT];
    double dt;
    const double *m_i;    /* nnodes      lumped nodal mass               */
    const double *vhat;   /* nnodes*3    inertia target v^n + dt g (amb-4)         */
    const uint8_t *freed; /* nnodes      1 = free DOF (m_i>0, not Dirichlet)      */
    const double *m_c;    /* ncells      cell mass (cells with m_c>0 are quadrature) */
    const double *V_ck;   /* nmat*ncells rest volume per material slot      */
    const double *S_ck;   /* nmat*ncells*9 stretch base S_{c,k} (row-major)  */
    int32_t psd;          /* 1: the Hessian's per-cell blocks K_c are PSD-projected  */
} orc_problem;

/* ------------------------------------------------------------------------ */
/* small dense 3x3 helpers                                                  */
/* ------------------------------------------------------------------------ */
static int64_t ncells(const orc_grid *g) { return (int64_t)g->n[0] * g->n[1] * g->n[2]; }
static int64_t nnodes(const orc_grid *g) { return (int64_t)(g->n[0] + 1) * (g->n[1] + 1) * (g->n[2] + 1); }
static int64_t cid(const orc_grid *g, int i, int j, int k) { return ((int64_t)i * g->n[1] + j) * g->n[2] + k; }
static int64_t nid(const orc_grid *g, int i, int j, int k) {
    return ((int64_t)i * (g->n[1] + 1) + j) * (g->n[2] + 1) + k;
}

static void mat_mul(const double A[9], const double B[9], double C[9]) {
    double T[9];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int e = 0; e < 3; e++) s += A[3 * a + e] * B[3 * e + b];
            T[3 * a + b] = s;
        }
    memcpy(C, T, sizeof T);
}
static void mat_T(const double A[9], double B[9]) {
    double T[9];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) T[3 * a + b] = A[3 * b + a];
    memcpy(B, T, sizeof T);
}
static double mat_det(const double A[9]) {
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}
/* inverse via adjugate / det */
static void mat_inv(const double A[9], double B[9]) {
    double d = mat_det(A), T[9];
    T[0] = (A[4] * A[8] - A[5] * A[7]) / d;
    T[1] = (A[2] * A[7] - A[1] * A[8]) / d;
    T[2] = (A[1] * A[5] - A[2] * A[4]) / d;
    T[3] = (A[5] * A[6] - A[3] * A[8]) / d;
    T[4] = (A[0] * A[8] - A[2] * A[6]) / d;
    T[5] = (A[2] * A[3] - A[0] * A[5]) / d;
    T[6] = (A[3] * A[7] - A[4] * A[6]) / d;
    T[7] = (A[1] * A[6] - A[0] * A[7]) / d;
    T[8] = (A[0] * A[4] - A[1] * A[3]) / d;
    memcpy(B, T, sizeof T);
}

/* Symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations (textbook):
 * A = Q diag(w) Q^T, columns of Q are eigenvectors.  Runs to convergence. */
void orc_sym_eig3(const double Ain[9], double w[3], double Q[9]) {
    double A[9];
    memcpy(A, Ain, sizeof A);
    for (int a = 0; a < 9; a++) Q[a] = (a % 4 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
        double dia = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
        if (off == 0.0 || off <= 1e-40 * dia) break;
        static const int PQ[3][2] = {{0, 1}, {0, 2}, {1, 2}};
        for (int r = 0; r < 3; r++) {
            int p = PQ[r][0], q = PQ[r][1];
            double apq = A[3 * p + q];
            if (apq == 0.0) continue;
            double theta = (A[3 * q + q] - A[3 * p + p]) / (2.0 * apq);
            double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
            double J[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, JT[9];
            J[3 * p + p] = c;
            J[3 * q + q] = c;
            J[3 * p + q] = s;
            J[3 * q + p] = -s;
            mat_T(J, JT);
            mat_mul(JT, A, A);
            mat_mul(A, J, A);
            mat_mul(Q, J, Q);
        }
    }
    for (int a = 0; a < 3; a++) w[a] = A[4 * a];
}

static void lame(const orc_material *m, double *mu, double *lam) {
    /* amb-2: standard 3D Lame parameters from (E, nu) */
    *mu = m->E / (2.0 * (1.0 + m->nu));
    *lam = m->E * m->nu / ((1.0 + m->nu) * (1.0 - 2.0 * m->nu));
}

/* ------------------------------------------------------------------------ */
/* C1: Q1 particle -> centre weights ("w_cp = N_c(x_p)"; App. A) */
/* ------------------------------------------------------------------------ */
/* base cell b = floor((x-o)/dx - 1/2), fraction f in [0,1); the 2^3 stencil cells are b+o */
void orc_base_cell(const orc_grid *g, const double x[3], int32_t b[3], double f[3]) {
    for (int a = 0; a < 3; a++) {
        double t = (x[a] - g->origin[a]) / g->dx - 0.5;
        double fb = floor(t);
        b[a] = (int32_t)fb;
        f[a] = t - fb;
    }
}
/* tensor-product tent evaluated at x for the 8 centres: w = prod_a (o_a ? f_a : 1 - f_a) */
void orc_q1_weights(const double f[3], double w[8]) {
    for (int o = 0; o < 8; o++) {
        int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
        w[o] = (ox ? f[0] : 1.0 - f[0]) * (oy ? f[1] : 1.0 - f[1]) * (oz ? f[2] : 1.0 - f[2]);
    }
}
/* centre -> node gradient: grad w_ic = (x_i - x_c)/(2^{d-2} dx^2), d = 3 */
static void grad_w(const orc_grid *g, int o, double gw[3]) {
    int oo[3] = {(o >> 2) & 1, (o >> 1) & 1, o & 1};
    for (int a = 0; a < 3; a++) {
        double xi_minus_xc = g->dx * (oo[a] - 0.5);
        gw[a] = xi_minus_xc / (2.0 * g->dx * g->dx);
    }
}

int orc_base_cells(const orc_grid *g, int64_t np, const double *x, int32_t *base) {
    for (int64_t p = 0; p < np; p++) {
        double f[3];
        orc_base_cell(g, x + 3 * p, base + 3 * p, f);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C2: StVK-Hencky Kirchhoff stress (P:172-178 Eq. spectral-map; P:200-205   */
/* Eq. hencky-taui): tau_i = 2 mu log sigma_i + lam sum_j log sigma_j, in the */
/* eigenbasis of b = F F^T (sigma_i^2 = beta_i).  b - I is formed as          */
/* H + H^T + H H^T (H = F - I) and log beta = log1p(eig(b - I)).              */
/* ------------------------------------------------------------------------ */
int orc_hencky_tau(const double F[9], double mu, double lam, double tau[9]) {
    if (!(mat_det(F) > 0.0)) return -1; /* inverted element */
    double H[9], HT[9], HHT[9], Bm[9], w[3], Q[9];
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? 1.0 : 0.0);
    mat_T(H, HT);
    mat_mul(H, HT, HHT);
    for (int a = 0; a < 9; a++) Bm[a] = H[a] + HT[a] + HHT[a];
    orc_sym_eig3(Bm, w, Q);
    double e[3], tr = 0;
    for (int i = 0; i < 3; i++) {
        e[i] = 0.5 * log1p(w[i]); /* log sigma_i = (1/2) log beta_i */
        tr += e[i];
    }
    double ti[3];
    for (int i = 0; i < 3; i++) ti[i] = 2.0 * mu * e[i] + lam * tr;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double s = 0;
            for (int i = 0; i < 3; i++) s += Q[3 * a + i] * ti[i] * Q[3 * b + i];
            tau[3 * a + b] = s;
        }
    return 0;
}

/* StVK-Hencky energy density psi = mu sum (log sigma)^2 + lam/2 (sum log sigma)^2
 * (P:192-195 Eq. hencky-energy), evaluated from b - I as above. */
static double hencky_psi(const double F[9], double mu, double lam) {
    double H[9], HT[9], HHT[9], Bm[9], w[3], Q[9];
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? 1.0 : 0.0);
    mat_T(H, HT);
    mat_mul(H, HT, HHT);
    for (int a = 0; a < 9; a++) Bm[a] = H[a] + HT[a] + HHT[a];
    orc_sym_eig3(Bm, w, Q);
    double s2 = 0, tr = 0;
    for (int i = 0; i < 3; i++) {
        double e = 0.5 * log1p(w[i]);
        s2 += e * e;
        tr += e;
    }
    return mu * s2 + 0.5 * lam * tr * tr;
}

double orc_hencky_psi(const double F[9], double mu, double lam) { return hencky_psi(F, mu, lam); }

/* ------------------------------------------------------------------------ */
/* Split Neo-Hookean (§4.3.2, d = 3):                              */
/*   Psi(F) = mu/2 (tr((J^{-1/3}F)^T (J^{-1/3}F)) - 3) + kappa/4 (J^2 - 1 - 2 log J)   */
/*            (Eq. split-nh-energy; kappa = 2/3 mu + lam)                */
/*   tau(F) = mu J^{-2/3} dev(b) + alpha(J) I, alpha = kappa/2 (J^2 - 1)       */
/*            (Eq. split-nh-tau)                                     */
/* Written out as the paper states them (the oracle is fp64).                 */
/* ------------------------------------------------------------------------ */
static double nh_kappa(double mu, double lam) { return 2.0 * mu / 3.0 + lam; }

int orc_nh_tau(const double F[9], double mu, double kappa, double tau[9]) {
    double J = mat_det(F);
    if (!(J > 0.0)) return -1;
    double FT[9], b[9];
    mat_T(F, FT);
    mat_mul(F, FT, b);
    double trb = b[0] + b[4] + b[8];
    double Jm23 = pow(J, -2.0 / 3.0);
    double alpha = 0.5 * kappa * (J * J - 1.0);
    for (int a = 0; a < 9; a++) {
        double devb = b[a] - ((a % 4 == 0) ? trb / 3.0 : 0.0);
        tau[a] = mu * Jm23 * devb + ((a % 4 == 0) ? alpha : 0.0);
    }
    return 0;
}

double orc_nh_psi(const double F[9], double mu, double kappa) {
    double J = mat_det(F);
    if (!(J > 0.0)) return INFINITY;
    double FT[9], C[9];
    mat_T(F, FT);
    mat_mul(FT, F, C);
    double trC = C[0] + C[4] + C[8];
    return 0.5 * mu * (pow(J, -2.0 / 3.0) * trC - 3.0) + 0.25 * kappa * (J * J - 1.0 - 2.0 * log(J));
}

/* Directional derivative of tau along dF (differentiating Eq. split-nh-tau):
 *   dJ = J tr(F^{-1} dF); db = dF F^T + F dF^T;
 *   dtau = mu [ -2/3 J^{-2/3} (dJ/J) dev(b) + J^{-2/3} dev(db) ] + kappa J dJ I. */
static void nh_dtau(const double F[9], const double dF[9], double mu, double kappa, double dtau[9]) {
    double J = mat_det(F), Fi[9], FidF[9], FT[9], dFT[9], b[9], t1[9], t2[9], db[9];
    mat_inv(F, Fi);
    mat_mul(Fi, dF, FidF);
    double dJ = J * (FidF[0] + FidF[4] + FidF[8]);
    mat_T(F, FT);
    mat_T(dF, dFT);
    mat_mul(F, FT, b);
    mat_mul(dF, FT, t1);
    mat_mul(F, dFT, t2);
    for (int a = 0; a < 9; a++) db[a] = t1[a] + t2[a];
    double trb = b[0] + b[4] + b[8], trdb = db[0] + db[4] + db[8];
    double Jm23 = pow(J, -2.0 / 3.0);
    for (int a = 0; a < 9; a++) {
        double dev_b = b[a] - ((a % 4 == 0) ? trb / 3.0 : 0.0);
        double dev_db = db[a] - ((a % 4 == 0) ? trdb / 3.0 : 0.0);
        dtau[a] = mu * (-2.0 / 3.0 * Jm23 * (dJ / J) * dev_b + Jm23 * dev_db) + ((a % 4 == 0) ? kappa * J * dJ : 0.0);
    }
}

/* ------------------------------------------------------------------------ */
/* J-based water (§4.5):                                           */
/*   psi(J) = kappa/2 (J - 1)^2 ;  pi(J) = J psi'(J) = kappa J (J - 1) ;       */
/*   tau = pi I (the hydrostatic Kirchhoff stress; the particle carries only  */
/*   J = det F_p) ;  J_base = (1 + sqrt(1 + 4 pi_c / kappa)) / 2 (positive    */
/*   root; the radicand is clamped at 0, its minimum over J > 0 being 0 at J=1/2). */
/* kappa is the material's E ("we use E in place of kappa").          */
/* ------------------------------------------------------------------------ */
double orc_water_pi(double J, double kappa) { return kappa * J * (J - 1.0); }
double orc_water_psi_J(double J, double kappa) { return 0.5 * kappa * (J - 1.0) * (J - 1.0); }
double orc_water_jbase(double pi, double kappa) {
    double r = 1.0 + 4.0 * pi / kappa;
    if (r < 0.0) r = 0.0;
    return 0.5 * (1.0 + sqrt(r));
}
int orc_water_tau(const double F[9], double kappa, double tau[9]) {
    double J = mat_det(F);
    if (!(J > 0.0)) return -1;
    for (int a = 0; a < 9; a++) tau[a] = (a % 4 == 0) ? orc_water_pi(J, kappa) : 0.0;
    return 0;
}
double orc_water_psi(const double F[9], double kappa) {
    double J = mat_det(F);
    if (!(J > 0.0)) return INFINITY;
    return orc_water_psi_J(J, kappa);
}
/* d tau along dF: dJ = J tr(F^{-1} dF), d pi = kappa (2J - 1) dJ */
static void water_dtau(const double F[9], const double dF[9], double kappa, double dtau[9]) {
    double J = mat_det(F), Fi[9], FidF[9];
    mat_inv(F, Fi);
    mat_mul(Fi, dF, FidF);
    double dJ = J * (FidF[0] + FidF[4] + FidF[8]);
    for (int a = 0; a < 9; a++) dtau[a] = (a % 4 == 0) ? kappa * (2.0 * J - 1.0) * dJ : 0.0;
}
/* base stretch of a water slot: S = J_base^{1/3} I, pi_c = tr(tau_c)/3 (det S = J_base) */
void orc_water_stretch(const double tau[9], double kappa, double S[9]) {
    double Jb = orc_water_jbase((tau[0] + tau[4] + tau[8]) / 3.0, kappa);
    double s = cbrt(Jb);
    for (int a = 0; a < 9; a++) S[a] = (a % 4 == 0) ? s : 0.0;
}

/* Cardano root of m^3 + p m + q = 0 on the admissible branch m > -min_i delta_i (App. C,
 * P:1305-1348; Eqs. cardano-one-real / cardano-three-real).  *branch = 1 (Delta >= 0) or 3. */
static double cbrt_signed(double z) { return z < 0 ? -pow(-z, 1.0 / 3.0) : pow(z, 1.0 / 3.0); }
double orc_nh_cardano(double p, double q, double dmin, int32_t *branch) {
    double Delta = (q / 2.0) * (q / 2.0) + (p / 3.0) * (p / 3.0) * (p / 3.0);
    if (Delta >= 0.0) {
        if (branch) *branch = 1;
        /* m = cbrt(-q/2 + sqrt D) + cbrt(-q/2 - sqrt D) (Eq. cardano-one-real).  The two cube roots
         * u, v satisfy u v = -p/3; the one of larger magnitude is taken from the formula and the other
         * as -p/(3u) — the same expression without the cancellation of -q/2 - sqrt D when |p| << |q|. */
        double sd = sqrt(Delta);
        double u = cbrt_signed(-q / 2.0 + (q <= 0.0 ? sd : -sd));
        return u != 0.0 ? u - p / (3.0 * u) : 0.0;
    }
    if (branch) *branch = 3;
    double r = 2.0 * sqrt(-p / 3.0);
    double arg = (3.0 * q / (2.0 * p)) * sqrt(-3.0 / p);
    if (arg > 1.0) arg = 1.0; /* "we clamp the arccos argument in [-1,1]" */
    if (arg < -1.0) arg = -1.0;
    double theta = acos(arg) / 3.0;
    double best = NAN;
    for (int k = 0; k < 3; k++) { /* the admissible root: beta_i = m + delta_i > 0 for all i */
        double m = r * cos(theta - 2.0 * M_PI * k / 3.0);
        if (m > -dmin && (isnan(best) || m > best)) best = m;
    }
    return best;
}

/* Stretch reconstruction (§4.3.2 P:258-271 + App. C): tau = U diag(tau_i) U^T;
 * alpha = tr(tau)/3, J = sqrt(1 + 2 alpha / kappa) (Eq. J-from-alpha), s = mu J^{-2/3},
 * delta_i = (tau_i - alpha)/s, S2 = sum_{i<j} delta_i delta_j, S3 = prod delta_i; the cubic
 * m^3 + S2 m + (S3 - J^2) = 0 (Eq. m-3D), beta_i = m + delta_i, sigma_i = sqrt(beta_i),
 * S = U diag(sigma) U^T.  Returns -1 outside the inversion domain (1 + 2 alpha/kappa <= 0). */
int orc_nh_stretch(const double tau[9], double mu, double kappa, double S[9], int32_t *branch) {
    double w[3], U[9];
    orc_sym_eig3(tau, w, U);
    double alpha = (w[0] + w[1] + w[2]) / 3.0;
    double J2 = 1.0 + 2.0 * alpha / kappa;
    if (!(J2 > 0.0)) return -1;
    double J = sqrt(J2);
    double s = mu * pow(J, -2.0 / 3.0);
    double d[3];
    for (int i = 0; i < 3; i++) d[i] = (w[i] - alpha) / s;
    double S2 = d[0] * d[1] + d[1] * d[2] + d[2] * d[0], S3 = d[0] * d[1] * d[2];
    double dmin = fmin(d[0], fmin(d[1], d[2]));
    double m = orc_nh_cardano(S2, S3 - J * J, dmin, branch);
    /* The reconstruction is defined by the root of Eq. m-3D; Cardano's closed form (which picks the
     * admissible branch) loses digits near a double root, so the root is refined by Newton steps on
     * the same cubic (reading f1-a). */
    for (int it = 0; it < 3; it++) {
        double f = m * m * m + S2 * m + (S3 - J * J), df = 3.0 * m * m + S2;
        if (!(fabs(df) > 1e-300)) break;
        double mn = m - f / df;
        if (!(mn > -dmin)) break;
        m = mn;
    }
    double sig[3];
    for (int i = 0; i < 3; i++) {
        double beta = m + d[i];
        if (!(beta > 0.0)) return -1;
        sig[i] = sqrt(beta);
    }
    for (int a = 0; a < 3; a++)
        for (int b2 = 0; b2 < 3; b2++) {
            double v = 0;
            for (int i = 0; i < 3; i++) v += U[3 * a + i] * sig[i] * U[3 * b2 + i];
            S[3 * a + b2] = v;
        }
    return 0;
}

/* ---- per-material dispatch (each material slot keeps its own constitutive law) ---- */
static int law_tau(const orc_material *m, const double F[9], double tau[9]) {
    double mu, lam;
    if (m->kind == 2) return orc_water_tau(F, m->E, tau);
    lame(m, &mu, &lam);
    return m->kind == 1 ? orc_nh_tau(F, mu, nh_kappa(mu, lam), tau) : orc_hencky_tau(F, mu, lam, tau);
}
static double law_psi(const orc_material *m, const double F[9]) {
    double mu, lam;
    if (m->kind == 2) return orc_water_psi(F, m->E);
    lame(m, &mu, &lam);
    return m->kind == 1 ? orc_nh_psi(F, mu, nh_kappa(mu, lam)) : hencky_psi(F, mu, lam);
}

/* ------------------------------------------------------------------------ */
/* C3: particle -> quadrature unload (Alg. 2 lines 1-9; Eqs.        */
/* p2c-mV, p2c-mv-affine, p2c-A-sum P:64-68; Eq. vtau).  Outputs the   */
/* raw accumulators; orc_normalize performs Alg. 2 lines 10-15.                */
/* clip=1 silently drops stencil cells outside the grid (window mode);         */
/* clip=0 reports them as out-of-domain (returns -(p+1)).                      */
/* Returns -(p+1) also for det F_p <= 0.                                      */
/* ------------------------------------------------------------------------ */
int64_t orc_p2q(const orc_grid *g, int32_t nmat, const orc_material *mats, int64_t np,
                const double *x, const double *v, const double *F, const double *G,
                const double *vol, const int32_t *mat, int32_t clip,
                double *m_c, double *mv_c, double *mG_c, double *V_ck, double *Vtau_ck) {
    int64_t nc = ncells(g);
    memset(m_c, 0, sizeof(double) * nc);
    memset(mv_c, 0, sizeof(double) * nc * 3);
    memset(mG_c, 0, sizeof(double) * nc * 9);
    memset(V_ck, 0, sizeof(double) * nc * nmat);
    memset(Vtau_ck, 0, sizeof(double) * nc * nmat * 9);
    for (int64_t p = 0; p < np; p++) {
        int k = mat[p];
        if (k < 0 || k >= nmat) return -(p + 1);
        double mp = mats[k].rho * vol[p]; /* m_p = rho V_p */
        double tau[9];
        if (law_tau(&mats[k], F + 9 * p, tau)) return -(p + 1); /* Alg. 2 line 3 */
        int32_t b[3];
        double f[3], w[8];
        orc_base_cell(g, x + 3 * p, b, f);
        orc_q1_weights(f, w);
        for (int o = 0; o < 8; o++) {
            int ci = b[0] + ((o >> 2) & 1), cj = b[1] + ((o >> 1) & 1), ck = b[2] + (o & 1);
            if (ci < 0 || cj < 0 || ck < 0 || ci >= g->n[0] || cj >= g->n[1] || ck >= g->n[2]) {
                if (clip) continue;
                return -(p + 1);
            }
            int64_t c = cid(g, ci, cj, ck);
            double xc[3] = {g->origin[0] + g->dx * (ci + 0.5), g->origin[1] + g->dx * (cj + 0.5),
                            g->origin[2] + g->dx * (ck + 0.5)};
            double d[3] = {xc[0] - x[3 * p], xc[1] - x[3 * p + 1], xc[2] - x[3 * p + 2]};
            const double *Gp = G + 9 * p;
            m_c[c] += w[o] * mp;                                       /* Eq. p2c-mV        */
            for (int a = 0; a < 3; a++) {                              /* Eq. p2c-mv-affine */
                double gd = Gp[3 * a] * d[0] + Gp[3 * a + 1] * d[1] + Gp[3 * a + 2] * d[2];
                mv_c[3 * c + a] += w[o] * mp * (v[3 * p + a] + gd);
            }
            for (int a = 0; a < 9; a++) mG_c[9 * c + a] += w[o] * mp * Gp[a]; /* Eq. p2c-A-sum */
            V_ck[(int64_t)k * nc + c] += w[o] * vol[p];                        /* V_c = sum w V_p  */
            for (int a = 0; a < 9; a++)
                Vtau_ck[((int64_t)k * nc + c) * 9 + a] += w[o] * vol[p] * tau[a]; /* Eq. vtau */
        }
    }
    return 0;
}

/* Alg. 2 lines 10-15: v_c = (mv)_c/m_c, G_c = (mG)_c/m_c, tau_ck = (V tau)/V */
void orc_normalize(const orc_grid *g, int32_t nmat, const double *m_c, const double *mv_c,
                   const double *mG_c, const double *V_ck, const double *Vtau_ck, double *v_c,
                   double *G_c, double *tau_ck) {
    int64_t nc = ncells(g);
    for (int64_t c = 0; c < nc; c++) {
        for (int a = 0; a < 3; a++) v_c[3 * c + a] = m_c[c] != 0.0 ? mv_c[3 * c + a] / m_c[c] : 0.0;
        for (int a = 0; a < 9; a++) G_c[9 * c + a] = m_c[c] != 0.0 ? mG_c[9 * c + a] / m_c[c] : 0.0;
        for (int k = 0; k < nmat; k++) {
            double V = V_ck[(int64_t)k * nc + c];
            for (int a = 0; a < 9; a++)
                tau_ck[((int64_t)k * nc + c) * 9 + a] =
                    V != 0.0 ? Vtau_ck[((int64_t)k * nc + c) * 9 + a] / V : 0.0;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* C4: centre -> node gather with w_ic = 2^-d (Alg. 2 lines 16-21)   */
/*   m_i = sum_c w_ic m_c ; (mv)_i = sum_c w_ic m_c (v_c + G_c (x_i - x_c)) ;  */
/*   v_i = (mv)_i / m_i.                                                       */
/* ------------------------------------------------------------------------ */
void orc_c2n(const orc_grid *g, const double *m_c, const double *v_c, const double *G_c,
             double *m_i, double *v_i) {
    int64_t nn = nnodes(g);
    double *mv = (double *)calloc((size_t)nn * 3, sizeof(double));
    memset(m_i, 0, sizeof(double) * nn);
    for (int ci = 0; ci < g->n[0]; ci++)
        for (int cj = 0; cj < g->n[1]; cj++)
            for (int ck = 0; ck < g->n[2]; ck++) {
                int64_t c = cid(g, ci, cj, ck);
                if (m_c[c] == 0.0) continue;
                for (int o = 0; o < 8; o++) {
                    int oo[3] = {(o >> 2) & 1, (o >> 1) & 1, o & 1};
                    int64_t i = nid(g, ci + oo[0], cj + oo[1], ck + oo[2]);
                    double d[3] = {g->dx * (oo[0] - 0.5), g->dx * (oo[1] - 0.5), g->dx * (oo[2] - 0.5)};
                    const double wic = 1.0 / 8.0;
                    m_i[i] += wic * m_c[c];
                    for (int a = 0; a < 3; a++) {
                        const double *Gc = G_c + 9 * c;
                        double gd = Gc[3 * a] * d[0] + Gc[3 * a + 1] * d[1] + Gc[3 * a + 2] * d[2];
                        mv[3 * i + a] += wic * m_c[c] * (v_c[3 * c + a] + gd);
                    }
                }
            }
    for (int64_t i = 0; i < nn; i++)
        for (int a = 0; a < 3; a++) v_i[3 * i + a] = m_i[i] != 0.0 ? mv[3 * i + a] / m_i[i] : 0.0;
    free(mv);
}

/* Dirichlet projection sets (amb-9): node i is fixed when lo <= x_i <= hi in all axes for
 * some box; free DOFs are nodes with m_i > 0 that are not fixed.  vfix gets the box velocity. */
void orc_dirichlet(const orc_grid *g, int32_t nbox, const orc_box *boxes, const double *m_i,
                   uint8_t *freed, double *vfix) {
    for (int i = 0; i <= g->n[0]; i++)
        for (int j = 0; j <= g->n[1]; j++)
            for (int k = 0; k <= g->n[2]; k++) {
                int64_t id = nid(g, i, j, k);
                double xi[3] = {g->origin[0] + g->dx * i, g->origin[1] + g->dx * j, g->origin[2] + g->dx * k};
                int fixed = -1;
                for (int b = 0; b < nbox; b++) {
                    int in = 1;
                    for (int a = 0; a < 3; a++)
                        if (!(xi[a] >= boxes[b].lo[a] && xi[a] <= boxes[b].hi[a])) in = 0;
                    if (in) { fixed = b; break; }
                }
                freed[id] = (m_i[id] > 0.0 && fixed < 0) ? 1 : 0;
                for (int a = 0; a < 3; a++) vfix[3 * id + a] = fixed >= 0 ? boxes[fixed].vel[a] : 0.0;
            }
}

/* ------------------------------------------------------------------------ */
/* C5: rotation-free stretch reconstruction for StVK-Hencky (P:156-160       */
/* Eq. rotfree-def; P:206-226 Eqs. hencky-trace/ei/sigmai):        */
/*   tau = U diag(tau_i) U^T ; s = tr tau/(2 mu + d lam) ; e_i = (tau_i - lam s)/(2 mu) ; */
/*   S = U diag(exp(e_i)) U^T.                                               */
/* ------------------------------------------------------------------------ */
void orc_stretch(const double tau[9], double mu, double lam, double S[9]) {
    double w[3], U[9];
    orc_sym_eig3(tau, w, U);
    double s = (w[0] + w[1] + w[2]) / (2.0 * mu + 3.0 * lam);
    double sig[3];
    for (int i = 0; i < 3; i++) sig[i] = exp((w[i] - lam * s) / (2.0 * mu));
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double v = 0;
            for (int i = 0; i < 3; i++) v += U[3 * a + i] * sig[i] * U[3 * b + i];
            S[3 * a + b] = v;
        }
}

void orc_stretch_all(const orc_grid *g, int32_t nmat, const orc_material *mats, const double *V_ck,
                     const double *tau_ck, double *S_ck) {
    int64_t nc = ncells(g);
    for (int k = 0; k < nmat; k++) {
        double mu, lam;
        lame(&mats[k], &mu, &lam);
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < nc; c++) {
            double *S = S_ck + ((int64_t)k * nc + c) * 9;
            if (V_ck[(int64_t)k * nc + c] != 0.0) {
                const double *tau = tau_ck + ((int64_t)k * nc + c) * 9; /* Alg. 3 line 6 */
                if (mats[k].kind == 2) {
                    orc_water_stretch(tau, mats[k].E, S); /* Eq. J_base */
                } else if (mats[k].kind == 1) {
                    if (orc_nh_stretch(tau, mu, nh_kappa(mu, lam), S, NULL))
                        for (int a = 0; a < 9; a++) S[a] = NAN; /* outside the inversion domain */
                } else {
                    orc_stretch(tau, mu, lam, S);
                }
            } else
                for (int a = 0; a < 9; a++) S[a] = (a % 4 == 0) ? 1.0 : 0.0;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* C6: incremental potential, gradient, Hessian-vector product, Jacobi diagonal */
/* Phi(v) = sum_i 1/2 m_i |v_i - vhat_i|^2 + sum_{c,k} V_ck psi_k((I + dt G_c(v)) S_ck) */
/* (P:146-153 Eq. incpot-rotfree; Alg. 3 line 8 P:395; App. B Eq. Phi). */
/* ------------------------------------------------------------------------ */

/* G_c(v) = sum_{i in corners(c)} v_i (x) grad w_ic */
static void cell_G(const orc_problem *P, const double *v, int ci, int cj, int ck, double Gc[9]) {
    const orc_grid *g = &P->g;
    memset(Gc, 0, sizeof(double) * 9);
    for (int o = 0; o < 8; o++) {
        int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
        double gw[3];
        grad_w(g, o, gw);
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) Gc[3 * a + b] += v[3 * i + a] * gw[b];
    }
}

double orc_energy(const orc_problem *P, const double *v) {
    const orc_grid *g = &P->g;
    int64_t nn = nnodes(g), nc = ncells(g);
    double E = 0.0;
    for (int64_t i = 0; i < nn; i++) {
        if (P->m_i[i] == 0.0) continue;
        double d2 = 0;
        for (int a = 0; a < 3; a++) d2 += (v[3 * i + a] - P->vhat[3 * i + a]) * (v[3 * i + a] - P->vhat[3 * i + a]);
        E += 0.5 * P->m_i[i] * d2;
    }
    /* elastic part: one partial sum per x-slice of cells, added in slice order */
    double *part = calloc((size_t)g->n[0], sizeof(double));
    int inverted = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : inverted)
    for (int ci = 0; ci < g->n[0]; ci++)
        for (int cj = 0; cj < g->n[1]; cj++)
            for (int ck = 0; ck < g->n[2]; ck++) {
                int64_t c = cid(g, ci, cj, ck);
                if (P->m_c[c] == 0.0) continue;
                double Gc[9], A[9];
                cell_G(P, v, ci, cj, ck, Gc);
                for (int a = 0; a < 9; a++) A[a] = ((a % 4 == 0) ? 1.0 : 0.0) + P->dt * Gc[a];
                if (!(mat_det(A) > 0.0)) { inverted = 1; continue; } /* amb-21 */
                for (int k = 0; k < P->nmat; k++) {
                    double V = P->V_ck[(int64_t)k * nc + c];
                    if (V == 0.0) continue;
                    double F[9];
                    mat_mul(A, P->S_ck + ((int64_t)k * nc + c) * 9, F); /* Eq. Ftrial-rotfree */
                    part[ci] += V * law_psi(&P->mats[k], F);
                }
            }
    for (int ci = 0; ci < g->n[0]; ci++) E += part[ci];
    free(part);
    return inverted ? INFINITY : E;
}

/* Per-cell, per-slot gradient block: dt V tau(F) A^{-T}  (== dt V P(F) S^T, amb-3) */
static void slot_grad(double dt, double V, const orc_material *m, const double A[9], const double S[9],
                      double out[9]) {
    double F[9], tau[9], Ai[9], AiT[9];
    mat_mul(A, S, F);
    law_tau(m, F, tau);
    mat_inv(A, Ai);
    mat_T(Ai, AiT);
    mat_mul(tau, AiT, out);
    for (int a = 0; a < 9; a++) out[a] *= dt * V;
}

/* Daleckii-Krein divided difference of log (amb-20): L(x,y) = (log x - log y)/(x - y),
 * L(x,x) = 1/x, computed stably from the eigenvalues lx = x-1, ly = y-1 of b - I. */
static double dlog(double lx, double ly) {
    double y = 1.0 + ly;
    double t = (lx - ly) / y;
    if (fabs(t) < 1e-4) return (1.0 - t / 2.0 + t * t / 3.0 - t * t * t / 4.0) / y;
    return log1p(t) / (lx - ly);
}

/* Directional derivative of dt V tau(F) A^{-T} along dG (the tangent map K_c:dG of one slot):
 *   dF = dt dG S ; db = dF F^T + F dF^T ; D = Q (L o (Q^T db Q)) Q^T  (Daleckii-Krein) ;
 *   dtau = mu D + lam/2 tr(D) I ;  d(A^{-T}) = -A^{-T} (dt dG)^T A^{-T} ;
 *   out = dt V (dtau A^{-T} + tau d(A^{-T})).   (App. B; C6 of SURVEY §8(c)) */
static void slot_tangent(double dt, double V, const orc_material *m, const double A[9], const double S[9],
                         const double dG[9], double out[9]) {
    double mu, lam;
    lame(m, &mu, &lam);
    double F[9], H[9], HT[9], HHT[9], Bm[9], w[3], Q[9], QT[9];
    mat_mul(A, S, F);
    for (int a = 0; a < 9; a++) H[a] = F[a] - ((a % 4 == 0) ? 1.0 : 0.0);
    mat_T(H, HT);
    mat_mul(H, HT, HHT);
    for (int a = 0; a < 9; a++) Bm[a] = H[a] + HT[a] + HHT[a];
    orc_sym_eig3(Bm, w, Q);
    mat_T(Q, QT);
    double tau[9];
    orc_hencky_tau(F, mu, lam, tau);
    double dF[9], FT[9], dFT[9], t1[9], t2[9], db[9];
    mat_mul(dG, S, dF);
    for (int a = 0; a < 9; a++) dF[a] *= dt;
    mat_T(F, FT);
    mat_T(dF, dFT);
    mat_mul(dF, FT, t1);
    mat_mul(F, dFT, t2);
    for (int a = 0; a < 9; a++) db[a] = t1[a] + t2[a];
    double dbp[9], Dp[9], D[9];
    mat_mul(QT, db, dbp);
    mat_mul(dbp, Q, dbp);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) Dp[3 * i + j] = dlog(w[i], w[j]) * dbp[3 * i + j];
    mat_mul(Q, Dp, D);
    mat_mul(D, QT, D);
    double trD = D[0] + D[4] + D[8];
    double dtau[9];
    for (int a = 0; a < 9; a++) dtau[a] = mu * D[a] + ((a % 4 == 0) ? 0.5 * lam * trD : 0.0);
    if (m->kind == 1) { /* split Neo-Hookean: tau and its derivative directly (Eq. split-nh-tau) */
        orc_nh_tau(F, mu, nh_kappa(mu, lam), tau);
        nh_dtau(F, dF, mu, nh_kappa(mu, lam), dtau);
    } else if (m->kind == 2) { /* water: tau = pi(J) I */
        orc_water_tau(F, m->E, tau);
        water_dtau(F, dF, m->E, dtau);
    }
    double Ai[9], AiT[9], dGT[9], dAiT[9], r1[9], r2[9];
    mat_inv(A, Ai);
    mat_T(Ai, AiT);
    mat_T(dG, dGT);
    mat_mul(AiT, dGT, dAiT);
    mat_mul(dAiT, AiT, dAiT);
    for (int a = 0; a < 9; a++) dAiT[a] *= -dt;
    mat_mul(dtau, AiT, r1);
    mat_mul(tau, dAiT, r2);
    for (int a = 0; a < 9; a++) out[a] = dt * V * (r1[a] + r2[a]);
}

static void cell_A(const orc_problem *P, const double *v, int ci, int cj, int ck, double A[9]) {
    double Gc[9];
    cell_G(P, v, ci, cj, ck, Gc);
    for (int a = 0; a < 9; a++) A[a] = ((a % 4 == 0) ? 1.0 : 0.0) + P->dt * Gc[a];
}

/* g_i = m_i (v_i - vhat_i) + sum_c sum_k [dt V_ck tau_k A_c^{-T}] grad w_ic (App. B Eq. residual,
 * P:1167-1175, with the sign of amb-3).  Written for all nodes; rows with m_i = 0 stay 0. */
void orc_gradient(const orc_problem *P, const double *v, double *grad) {
    const orc_grid *g = &P->g;
    int64_t nn = nnodes(g), nc = ncells(g);
    for (int64_t i = 0; i < nn; i++)
        for (int a = 0; a < 3; a++)
            grad[3 * i + a] = P->m_i[i] != 0.0 ? P->m_i[i] * (v[3 * i + a] - P->vhat[3 * i + a]) : 0.0;
    for (int col = 0; col < 8; col++) /* cells of one colour share no node */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int ci = (col >> 2) & 1; ci < g->n[0]; ci += 2)
        for (int cj = (col >> 1) & 1; cj < g->n[1]; cj += 2)
            for (int ck = col & 1; ck < g->n[2]; ck += 2) {
                int64_t c = cid(g, ci, cj, ck);
                if (P->m_c[c] == 0.0) continue;
                double A[9], Pc[9] = {0};
                cell_A(P, v, ci, cj, ck, A);
                for (int k = 0; k < P->nmat; k++) {
                    double V = P->V_ck[(int64_t)k * nc + c];
                    if (V == 0.0) continue;
                    double blk[9];
                    slot_grad(P->dt, V, &P->mats[k], A, P->S_ck + ((int64_t)k * nc + c) * 9, blk);
                    for (int a = 0; a < 9; a++) Pc[a] += blk[a];
                }
                for (int o = 0; o < 8; o++) {
                    int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
                    double gw[3];
                    grad_w(g, o, gw);
                    for (int a = 0; a < 3; a++)
                        grad[3 * i + a] += Pc[3 * a] * gw[0] + Pc[3 * a + 1] * gw[1] + Pc[3 * a + 2] * gw[2];
                }
            }
}

/* Per-cell PSD projection ("per-cell PSD projection of the elastic energy Hessian
 * (eigenvalue clamping at 0)"): M -> Q max(Lambda, 0) Q^T for a symmetric 9x9 M, eigenpairs by the
 * textbook cyclic Jacobi method (rotations until the off-diagonal part vanishes). */
void orc_psd_project9(const double Min[81], double Mout[81]) {
    double A[81], V[81];
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++) {
            A[9 * r + c] = 0.5 * (Min[9 * r + c] + Min[9 * c + r]);
            V[9 * r + c] = (r == c) ? 1.0 : 0.0;
        }
    for (int sweep = 0; sweep < 50; sweep++) {
        double off = 0.0, dg = 0.0;
        for (int r = 0; r < 9; r++)
            for (int c = 0; c < 9; c++) {
                if (r != c) off += A[9 * r + c] * A[9 * r + c];
                else dg += A[9 * r + c] * A[9 * r + c];
            }
        if (!(off > 1e-32 * dg)) break;
        for (int p = 0; p < 8; p++)
            for (int q = p + 1; q < 9; q++) {
                double apq = A[9 * p + q];
                if (apq == 0.0) continue;
                double theta = (A[9 * q + q] - A[9 * p + p]) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int r = 0; r < 9; r++) { /* columns p, q */
                    double arp = A[9 * r + p], arq = A[9 * r + q];
                    A[9 * r + p] = c * arp - s * arq;
                    A[9 * r + q] = s * arp + c * arq;
                }
                for (int r = 0; r < 9; r++) { /* rows p, q */
                    double apr = A[9 * p + r], aqr = A[9 * q + r];
                    A[9 * p + r] = c * apr - s * aqr;
                    A[9 * q + r] = s * apr + c * aqr;
                }
                for (int r = 0; r < 9; r++) { /* eigenvectors */
                    double vrp = V[9 * r + p], vrq = V[9 * r + q];
                    V[9 * r + p] = c * vrp - s * vrq;
                    V[9 * r + q] = s * vrp + c * vrq;
                }
            }
    }
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++) {
            double v = 0.0;
            for (int i = 0; i < 9; i++) {
                double l = A[9 * i + i] > 0.0 ? A[9 * i + i] : 0.0;
                v += V[9 * r + i] * l * V[9 * c + i];
            }
            Mout[9 * r + c] = v;
        }
}

/* The cell's tangent as a 9x9 matrix: column (e,f) = sum_k slot_tangent along the unit dG = e_e (x) e_f,
 * i.e. K_c[(a,b),(e,f)] = d Pc_ab / d G_ef with Pc = sum_k dt V tau A^{-T}; PSD-projected if P->psd. */
static void cell_tangent_matrix(const orc_problem *P, const double A[9], int64_t c, double M[81]) {
    int64_t nc = ncells(&P->g);
    for (int e = 0; e < 9; e++) {
        double dG[9] = {0}, Pc[9] = {0};
        dG[e] = 1.0;
        for (int k = 0; k < P->nmat; k++) {
            double V = P->V_ck[(int64_t)k * nc + c];
            if (V == 0.0) continue;
            double blk[9];
            slot_tangent(P->dt, V, &P->mats[k], A, P->S_ck + ((int64_t)k * nc + c) * 9, dG, blk);
            for (int a = 0; a < 9; a++) Pc[a] += blk[a];
        }
        for (int a = 0; a < 9; a++) M[9 * a + e] = Pc[a];
    }
    if (P->psd) orc_psd_project9(M, M);
}

/* (H u)_i = m_i u_i + sum_c [sum_k K_ck : dG_c(u)] grad w_ic,  dG_c(u) = sum_j u_j (x) grad w_jc
 * (Hessian of Phi at v, App. B; full, unprojected). */
void orc_hvp(const orc_problem *P, const double *v, const double *u, double *Hu) {
    const orc_grid *g = &P->g;
    int64_t nn = nnodes(g), nc = ncells(g);
    for (int64_t i = 0; i < nn; i++)
        for (int a = 0; a < 3; a++) Hu[3 * i + a] = P->m_i[i] != 0.0 ? P->m_i[i] * u[3 * i + a] : 0.0;
    for (int col = 0; col < 8; col++) /* cells of one colour share no node */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int ci = (col >> 2) & 1; ci < g->n[0]; ci += 2)
        for (int cj = (col >> 1) & 1; cj < g->n[1]; cj += 2)
            for (int ck = col & 1; ck < g->n[2]; ck += 2) {
                int64_t c = cid(g, ci, cj, ck);
                if (P->m_c[c] == 0.0) continue;
                double A[9], dG[9], Pc[9] = {0};
                cell_A(P, v, ci, cj, ck, A);
                cell_G(P, u, ci, cj, ck, dG);
                if (P->psd) { /* projected block: Pc = K_c^+ : dG */
                    double M[81];
                    cell_tangent_matrix(P, A, c, M);
                    for (int a = 0; a < 9; a++)
                        for (int e = 0; e < 9; e++) Pc[a] += M[9 * a + e] * dG[e];
                } else
                for (int k = 0; k < P->nmat; k++) {
                    double V = P->V_ck[(int64_t)k * nc + c];
                    if (V == 0.0) continue;
                    double blk[9];
                    slot_tangent(P->dt, V, &P->mats[k], A, P->S_ck + ((int64_t)k * nc + c) * 9, dG, blk);
                    for (int a = 0; a < 9; a++) Pc[a] += blk[a];
                }
                for (int o = 0; o < 8; o++) {
                    int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
                    double gw[3];
                    grad_w(g, o, gw);
                    for (int a = 0; a < 3; a++)
                        Hu[3 * i + a] += Pc[3 * a] * gw[0] + Pc[3 * a + 1] * gw[1] + Pc[3 * a + 2] * gw[2];
                }
            }
}

/* Jacobi diagonal (amb-8): D_ia = e_ia^T H e_ia = m_i + sum_c [K_c : (e_a (x) grad w_ic)] . e_a grad w_ic */
void orc_diag(const orc_problem *P, const double *v, double *D) {
    const orc_grid *g = &P->g;
    int64_t nn = nnodes(g), nc = ncells(g);
    for (int64_t i = 0; i < nn; i++)
        for (int a = 0; a < 3; a++) D[3 * i + a] = P->m_i[i];
    for (int col = 0; col < 8; col++) /* cells of one colour share no node */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int ci = (col >> 2) & 1; ci < g->n[0]; ci += 2)
        for (int cj = (col >> 1) & 1; cj < g->n[1]; cj += 2)
            for (int ck = col & 1; ck < g->n[2]; ck += 2) {
                int64_t c = cid(g, ci, cj, ck);
                if (P->m_c[c] == 0.0) continue;
                double A[9], M[81];
                cell_A(P, v, ci, cj, ck, A);
                if (P->psd) cell_tangent_matrix(P, A, c, M);
                for (int o = 0; o < 8; o++) {
                    int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
                    double gw[3];
                    grad_w(g, o, gw);
                    for (int a = 0; a < 3; a++) {
                        double dG[9] = {0}, Pc[9] = {0};
                        for (int b = 0; b < 3; b++) dG[3 * a + b] = gw[b];
                        if (P->psd) {
                            for (int r = 0; r < 9; r++)
                                for (int e = 0; e < 9; e++) Pc[r] += M[9 * r + e] * dG[e];
                        } else
                        for (int k = 0; k < P->nmat; k++) {
                            double V = P->V_ck[(int64_t)k * nc + c];
                            if (V == 0.0) continue;
                            double blk[9];
                            slot_tangent(P->dt, V, &P->mats[k], A, P->S_ck + ((int64_t)k * nc + c) * 9, dG, blk);
                            for (int e = 0; e < 9; e++) Pc[e] += blk[e];
                        }
                        D[3 * i + a] += Pc[3 * a] * gw[0] + Pc[3 * a + 1] * gw[1] + Pc[3 * a + 2] * gw[2];
                    }
                }
            }
}

/* ------------------------------------------------------------------------ */
/* C7: Newton with Jacobi-PCG and Armijo backtracking ("any standard */
/* solvers"; "preconditioned matrix-free conjugate gradient"    */
/* "damping/line-search").  Exact reading: amb-6, amb-7, amb-8. */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t newton_max, cg_max, ls_max;
    double eps_newton, eps_cg, armijo;
    int32_t fixed_newton; /* >0: run exactly this many Newton iterations              */
    const int32_t *fixed_cg; /* NULL or per-Newton-iteration CG iteration counts       */
    const int32_t *fixed_ls; /* NULL or per-Newton-iteration line-search halvings      */
    double ls_slack;         /* Armijo slack: accept when Phi_new <= Phi + c a g.p + slack |Phi| */
} orc_solver_cfg;

typedef struct {
    int32_t newton_iters, cg_total, ls_halvings, converged, neg_curv;
    double grad_norm0, grad_norm, energy;
    int32_t cg_iters[64];
    int32_t ls_iters[64];
} orc_solve_stats;

static double dotf(int64_t n, const uint8_t *fr, const double *a, const double *b) {
    /* fixed chunks of nodes, partial sums added in chunk order */
    const int64_t CH = 4096, nch = (n + CH - 1) / CH;
    double *part = calloc((size_t)(nch > 0 ? nch : 1), sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nch; q++) {
        double s = 0;
        for (int64_t i = q * CH; i < n && i < (q + 1) * CH; i++)
            if (fr[i])
                for (int c = 0; c < 3; c++) s += a[3 * i + c] * b[3 * i + c];
        part[q] = s;
    }
    double s = 0;
    for (int64_t q = 0; q < nch; q++) s += part[q];
    free(part);
    return s;
}

/* PCG on H p = -g over free DOFs; x0 = 0; stop ||r|| <= eps ||r0|| or it_max (or fixed count). */
static int pcg(const orc_problem *P, const double *v, const double *grad, const double *D, int it_max,
               double eps, int fixed, double *x, int *neg) {
    int64_t nn = nnodes(&P->g);
    const uint8_t *fr = P->freed;
    double *r = calloc(nn * 3, sizeof(double)), *z = calloc(nn * 3, sizeof(double));
    double *p = calloc(nn * 3, sizeof(double)), *Hp = calloc(nn * 3, sizeof(double));
    for (int64_t i = 0; i < nn * 3; i++) {
        int64_t n = i / 3;
        x[i] = 0.0;
        r[i] = fr[n] ? -grad[i] : 0.0;
        z[i] = fr[n] ? r[i] / D[i] : 0.0;
        p[i] = z[i];
    }
    double rz = dotf(nn, fr, r, z);
    double r0 = sqrt(dotf(nn, fr, r, r));
    int it = 0;
    *neg = 0;
    if (r0 == 0.0) goto done;
    for (it = 0; it < it_max;) {
        orc_hvp(P, v, p, Hp);
        double pHp = dotf(nn, fr, p, Hp);
        if (!(pHp > 0.0)) {
            *neg = 1;
            if (it == 0)
                for (int64_t i = 0; i < nn * 3; i++) x[i] = p[i];
            it++;
            break;
        }
        double alpha = rz / pHp;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nn * 3; i++)
            if (fr[i / 3]) {
                x[i] += alpha * p[i];
                r[i] -= alpha * Hp[i];
            }
        it++;
        double rn = sqrt(dotf(nn, fr, r, r));
        if (!fixed && rn <= eps * r0) break;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nn * 3; i++) z[i] = fr[i / 3] ? r[i] / D[i] : 0.0;
        double rz_new = dotf(nn, fr, r, z);
        double beta = rz_new / rz;
        rz = rz_new;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nn * 3; i++) p[i] = fr[i / 3] ? z[i] + beta * p[i] : 0.0;
    }
done:
    free(r); free(z); free(p); free(Hp);
    return it;
}

/* v (in/out): on entry the inertia target with Dirichlet values imposed on fixed nodes (v^0);
 * on return v^{n+1}. */
int64_t orc_plastic_update(const orc_problem *P, const double *v, const double *S_base, double *S_out);
static int any_plastic(const orc_problem *P);
int orc_newton(const orc_problem *P0, const orc_solver_cfg *cfg, double *v, orc_solve_stats *st) {
    int64_t nn = nnodes(&P0->g);
    const uint8_t *fr = P0->freed;
    double *grad = calloc(nn * 3, sizeof(double)), *D = calloc(nn * 3, sizeof(double));
    double *p = calloc(nn * 3, sizeof(double)), *vt = calloc(nn * 3, sizeof(double));
    memset(st, 0, sizeof *st);
    /* fixed-point plasticity: the bases are re-projected at every Newton iterate from S_base
     * and held fixed through that iteration's PCG and line search */
    const int plastic = any_plastic(P0);
    orc_problem Pw = *P0;
    double *S_work = NULL;
    if (plastic) {
        S_work = malloc(sizeof(double) * 9 * ncells(&P0->g) * P0->nmat);
        Pw.S_ck = S_work;
    }
    const orc_problem *P = &Pw;
    int kmax = cfg->fixed_newton > 0 ? cfg->fixed_newton : cfg->newton_max;
    for (int k = 0; k < kmax; k++) {
        if (plastic) orc_plastic_update(P0, v, P0->S_ck, S_work);
        orc_gradient(P, v, grad);
        double gn = sqrt(dotf(nn, fr, grad, grad));
        if (k == 0) st->grad_norm0 = gn;
        st->grad_norm = gn;
        if (cfg->fixed_newton <= 0 && gn <= cfg->eps_newton * st->grad_norm0) {
            st->converged = 1;
            break;
        }
        orc_diag(P, v, D);
        int neg = 0;
        int itmax = (cfg->fixed_cg != NULL) ? cfg->fixed_cg[k] : cfg->cg_max;
        int its = pcg(P, v, grad, D, itmax, cfg->eps_cg, cfg->fixed_cg != NULL, p, &neg);
        if (k < 64) st->cg_iters[k] = its;
        st->cg_total += its;
        st->neg_curv += neg;
        /* Armijo backtracking: alpha = 1, halve while Phi(v + alpha p) > Phi(v) + c alpha g.p */
        double phi0 = orc_energy(P, v), gp = dotf(nn, fr, grad, p), alpha = 1.0;
        int h = 0;
        if (cfg->fixed_ls != NULL) { /* parity replay of the halving count */
            for (h = 0; h < cfg->fixed_ls[k]; h++) alpha *= 0.5;
            for (int64_t i = 0; i < nn * 3; i++) vt[i] = fr[i / 3] ? v[i] + alpha * p[i] : v[i];
        } else {
            for (;;) {
                for (int64_t i = 0; i < nn * 3; i++) vt[i] = fr[i / 3] ? v[i] + alpha * p[i] : v[i];
                double phi = orc_energy(P, vt);
                /* Armijo with a rounding slack (amb-6): a decrease below the resolution of Phi
                 * cannot be measured, so it is not demanded. */
                if (phi <= phi0 + cfg->armijo * alpha * gp + cfg->ls_slack * fabs(phi0)) break;
                if (h >= cfg->ls_max) break; /* stagnation: accept */
                alpha *= 0.5;
                h++;
            }
        }
        if (k < 64) st->ls_iters[k] = h;
        st->ls_halvings += h;
        memcpy(v, vt, sizeof(double) * nn * 3);
        st->newton_iters = k + 1;
    }
    if (cfg->fixed_newton <= 0 && st->newton_iters == kmax && !st->converged) {
        if (plastic) orc_plastic_update(P0, v, P0->S_ck, S_work);
        orc_gradient(P, v, grad);
        st->grad_norm = sqrt(dotf(nn, fr, grad, grad));
        if (st->grad_norm <= cfg->eps_newton * st->grad_norm0) st->converged = 1;
    }
    st->energy = orc_energy(P, v);
    free(grad); free(D); free(p); free(vt); free(S_work);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Fixed-point plasticity (§6.5): von Mises return map in Hencky strain */
/* space, applied to the trial deformation of each plastic slot at every     */
/* Newton iterate, "while the matrix-free conjugate gradient solve handles elasticity only".        */
/*   F = U diag(sigma) V^T, e = log sigma, e_dev = e - tr(e)/3;                                     */
/*   if ||2 mu e_dev|| > sqrt(2/3) sigma_y:  e_dev <- s e_dev, s = sqrt(2/3) sigma_y / (2 mu ||e_dev||) */
/*   F^E = U diag(exp(e^E)) V^T = F P,  P = V diag(exp((s - 1) e_dev)) V^T  (from C = F^T F = V sigma^2 V^T) */
/* The volume is kept (tr e unchanged; det P = 1).  Returns 1 if the state was projected.            */
/* ------------------------------------------------------------------------ */
int orc_vm_plastic_P(const double F[9], double mu, double sigma_y, double Pm[9]) {
    double FT[9], Cm[9], lam[3], V[9];
    mat_T(F, FT);
    mat_mul(FT, F, Cm);
    orc_sym_eig3(Cm, lam, V);
    double e[3], tr = 0.0;
    for (int i = 0; i < 3; i++) {
        e[i] = 0.5 * log(lam[i]);
        tr += e[i];
    }
    double ed[3], nrm = 0.0;
    for (int i = 0; i < 3; i++) {
        ed[i] = e[i] - tr / 3.0;
        nrm += ed[i] * ed[i];
    }
    nrm = sqrt(nrm);
    for (int a = 0; a < 9; a++) Pm[a] = (a % 4 == 0) ? 1.0 : 0.0;
    if (!(2.0 * mu * nrm > sqrt(2.0 / 3.0) * sigma_y)) return 0;
    double sc = sqrt(2.0 / 3.0) * sigma_y / (2.0 * mu * nrm);
    double d[3];
    for (int i = 0; i < 3; i++) d[i] = exp((sc - 1.0) * ed[i]);
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double v = 0.0;
            for (int i = 0; i < 3; i++) v += V[3 * a + i] * d[i] * V[3 * b + i];
            Pm[3 * a + b] = v;
        }
    return 1;
}

void orc_vm_return(const double F[9], double mu, double sigma_y, double FE[9]) {
    double Pm[9];
    orc_vm_plastic_P(F, mu, sigma_y, Pm);
    mat_mul(F, Pm, FE);
}

/* Plastic update of the bases at iterate v (the fixed point on F): for each plastic slot,
 * F^tr = A(v) S_base, F^E = Z(F^tr), and the slot's base becomes S = A(v)^{-1} F^E = S_base P, so that
 * A(v) S = F^E; elastic slots keep S_base.  Returns the number of projected slots. */
int64_t orc_plastic_update(const orc_problem *P, const double *v, const double *S_base, double *S_out) {
    const orc_grid *g = &P->g;
    int64_t nc = ncells(g), nproj = 0;
    memcpy(S_out, S_base, sizeof(double) * 9 * nc * P->nmat);
    for (int k = 0; k < P->nmat; k++) {
        const orc_material *m = &P->mats[k];
        if (m->kind != 0 || !(m->yield_stress > 0.0)) continue;
        double mu, lam;
        lame(m, &mu, &lam);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : nproj)
        for (int ci = 0; ci < g->n[0]; ci++)
            for (int cj = 0; cj < g->n[1]; cj++)
                for (int ck = 0; ck < g->n[2]; ck++) {
                    int64_t c = cid(g, ci, cj, ck);
                    if (P->m_c[c] == 0.0 || P->V_ck[(int64_t)k * nc + c] == 0.0) continue;
                    double Gc[9], A[9], Ftr[9], Pm[9];
                    cell_G(P, v, ci, cj, ck, Gc);
                    for (int a = 0; a < 9; a++) A[a] = ((a % 4 == 0) ? 1.0 : 0.0) + P->dt * Gc[a];
                    const double *Sb = S_base + ((int64_t)k * nc + c) * 9;
                    mat_mul(A, Sb, Ftr);
                    nproj += orc_vm_plastic_P(Ftr, mu, m->yield_stress, Pm);
                    mat_mul(Sb, Pm, S_out + ((int64_t)k * nc + c) * 9);
                }
    }
    return nproj;
}

static int any_plastic(const orc_problem *P) {
    for (int k = 0; k < P->nmat; k++)
        if (P->mats[k].kind == 0 && P->mats[k].yield_stress > 0.0) return 1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C8: load back to particles (Alg. 4; P:71-76 Eqs. vc2p, Gc2p;   */
/* P:105-109):  for m_c != 0: v_c = sum w_ic v_i, G_c = sum v_i (x) grad w_ic; */
/* v_p = sum w_cp v_c ; G_p = sum w_cp G_c (weights from x_p^n) ;             */
/* x_p += dt v_p ; F_p <- (I + dt G_p) F_p.   (v_c = G_c = 0 where m_c = 0)   */
/* ------------------------------------------------------------------------ */
/* Water particles (kind 2) carry only J_p: their F_p is J_p^{1/3} I, updated by
 * J_p^{n+1} = (1 + dt tr(G_p)) J_p^n (the trace form; G_p = sum_c w_cp G_c^{n+1}).
 * Plastic particles (kind 0, yield_stress > 0) take the von Mises return map of their trial F. */
int64_t orc_g2p_mat(const orc_grid *g, double dt, const double *m_c, const double *v_i, int64_t np,
                    double *x, double *v, double *F, double *G, const int32_t *mat, const orc_material *mats,
                    int32_t clip);
int64_t orc_g2p(const orc_grid *g, double dt, const double *m_c, const double *v_i, int64_t np,
                double *x, double *v, double *F, double *G, int32_t clip) {
    return orc_g2p_mat(g, dt, m_c, v_i, np, x, v, F, G, NULL, NULL, clip);
}
int64_t orc_g2p_mat(const orc_grid *g, double dt, const double *m_c, const double *v_i, int64_t np,
                    double *x, double *v, double *F, double *G, const int32_t *mat, const orc_material *mats,
                    int32_t clip) {
    int64_t nc = ncells(g);
    double *vc = calloc(nc * 3, sizeof(double)), *Gc = calloc(nc * 9, sizeof(double));
#pragma omp parallel for schedule(static)
    for (int ci = 0; ci < g->n[0]; ci++)
        for (int cj = 0; cj < g->n[1]; cj++)
            for (int ck = 0; ck < g->n[2]; ck++) {
                int64_t c = cid(g, ci, cj, ck);
                if (m_c[c] == 0.0) continue;
                for (int o = 0; o < 8; o++) {
                    int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
                    double gw[3];
                    grad_w(g, o, gw);
                    for (int a = 0; a < 3; a++) {
                        vc[3 * c + a] += (1.0 / 8.0) * v_i[3 * i + a];
                        for (int b = 0; b < 3; b++) Gc[9 * c + 3 * a + b] += v_i[3 * i + a] * gw[b];
                    }
                }
            }
    for (int64_t p = 0; p < np; p++) {
        int32_t b[3];
        double f[3], w[8], vp[3] = {0}, Gp[9] = {0};
        orc_base_cell(g, x + 3 * p, b, f);
        orc_q1_weights(f, w);
        for (int o = 0; o < 8; o++) {
            int ci = b[0] + ((o >> 2) & 1), cj = b[1] + ((o >> 1) & 1), ck = b[2] + (o & 1);
            if (ci < 0 || cj < 0 || ck < 0 || ci >= g->n[0] || cj >= g->n[1] || ck >= g->n[2]) {
                if (clip) continue;
                free(vc); free(Gc);
                return -(p + 1);
            }
            int64_t c = cid(g, ci, cj, ck);
            for (int a = 0; a < 3; a++) vp[a] += w[o] * vc[3 * c + a];
            for (int a = 0; a < 9; a++) Gp[a] += w[o] * Gc[9 * c + a];
        }
        double A[9], Fn[9];
        for (int a = 0; a < 9; a++) A[a] = ((a % 4 == 0) ? 1.0 : 0.0) + dt * Gp[a];
        if (mat && mats[mat[p]].kind == 0 && mats[mat[p]].yield_stress > 0.0) {
            /* plastic particle: F_p^{n+1} = Z((I + dt G_p) F_p) (same von Mises return map) */
            double Ftr[9], mu, lam;
            mat_mul(A, F + 9 * p, Ftr);
            lame(&mats[mat[p]], &mu, &lam);
            orc_vm_return(Ftr, mu, mats[mat[p]].yield_stress, Fn);
        } else if (mat && mats[mat[p]].kind == 2) {
            double Jn = (1.0 + dt * (Gp[0] + Gp[4] + Gp[8])) * mat_det(F + 9 * p);
            double s = cbrt(Jn);
            for (int a = 0; a < 9; a++) Fn[a] = (a % 4 == 0) ? s : 0.0;
        } else {
            mat_mul(A, F + 9 * p, Fn);
        }
        for (int a = 0; a < 3; a++) {
            x[3 * p + a] += dt * vp[a];
            v[3 * p + a] = vp[a];
        }
        memcpy(F + 9 * p, Fn, sizeof Fn);
        memcpy(G + 9 * p, Gp, sizeof Gp);
    }
    free(vc); free(Gc);
    return 0;
}

/* Explicit force of Eq. explicitforce: f_i = - sum_c sum_k V_ck tau_ck grad w_ic.
 * Used only as the special case C6-(vii): at G_c = 0, g = m (v - vhat) - dt f. */
void orc_explicit_force(const orc_grid *g, int32_t nmat, const double *m_c, const double *V_ck,
                        const double *tau_ck, double *f) {
    int64_t nn = nnodes(g), nc = ncells(g);
    memset(f, 0, sizeof(double) * nn * 3);
    for (int col = 0; col < 8; col++) /* cells of one colour share no node */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int ci = (col >> 2) & 1; ci < g->n[0]; ci += 2)
        for (int cj = (col >> 1) & 1; cj < g->n[1]; cj += 2)
            for (int ck = col & 1; ck < g->n[2]; ck += 2) {
                int64_t c = cid(g, ci, cj, ck);
                if (m_c[c] == 0.0) continue;
                double Vt[9] = {0};
                for (int k = 0; k < nmat; k++)
                    for (int a = 0; a < 9; a++)
                        Vt[a] += V_ck[(int64_t)k * nc + c] * tau_ck[((int64_t)k * nc + c) * 9 + a];
                for (int o = 0; o < 8; o++) {
                    int64_t i = nid(g, ci + ((o >> 2) & 1), cj + ((o >> 1) & 1), ck + (o & 1));
                    double gw[3];
                    grad_w(g, o, gw);
                    for (int a = 0; a < 3; a++) f[3 * i + a] -= Vt[3 * a] * gw[0] + Vt[3 * a + 1] * gw[1] + Vt[3 * a + 2] * gw[2];
                }
            }
}
