/*
 * tpo_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * fp64 CPU restatement of the reference so3tpo hot path
 * (/root/reference/proj/src/{wigner,sphere,cgtp,gtp,mtp,irreps,bench}.cpp),
 * Eigen-free, exported with a C ABI so that tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs can call it through
 * ctypes.  The product path (paper_2506_13523_b200/) never links or calls
 * this library; it is the parity checker, not the thing measured or shipped.
 *
 * Parity status: PINNED against the reference's own known-answer tests
 * (proj/tests/test_{wigner,sphere,cgtp,gtp,mtp,irreps,bench}.cpp,
 * proj/README.md:99-108) and independent oracles (sympy real_gaunt /
 * clebsch_gordan, scipy roots_legendre / lpmv) -- see tests/test_oracle_*.py.
 * The reference binary itself cannot be built here (Eigen 3 missing,
 * proj/CMakeLists.txt:14-23), see DESIGN.md.
 *
 * Conventions follow the reference exactly: flat
 * layout m=-l..l per degree, real CG with odd-parity Im rule, l=1 order
 * (y,z,x), no Condon-Shortley phase, MIMO L3 = 2L.
 *
 * Degree lists: every irreps argument is a list of degrees `ls[0..n)` with
 * multiplicity 1 each (single-copy entries), which covers every caller of
 * the hot path (proj/src/bench.cpp:18-21, proj/src/verify.cpp:53-63).
 */
#ifndef TPO_ORACLE_H
#define TPO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror proj exceptions) */
#define ORC_OK 0
#define ORC_EINVAL 1   /* std::invalid_argument */
#define ORC_ERANGE 2   /* std::out_of_range */
#define ORC_ERUNTIME 3 /* std::runtime_error / logic_error */
#define ORC_ECAP 4     /* caller buffer too small */

const char* orc_last_error(void);

/* ---- RNG (proj/src/irreps.cpp:78-83, proj/src/wigner.cpp:219-226) ---- */
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void* rng);
/* fresh std::normal_distribution per call, like IrrepVector::random */
void orc_rng_irrep_random(void* rng, int dim, double* out);
/* Rotation::random: quaternion from 4 gaussians (g++ evaluates the Eigen
 * Quaterniond(w,x,y,z) constructor arguments right-to-left), normalized */
void orc_rng_rotation(void* rng, double* R9);

/* ---- tables (proj/src/wigner.cpp) ---- */
double orc_cg_coefficient(int l1, int m1, int l2, int m2, int l3, int m3);
/* real_basis_change(l): (2l+1)^2 complex, row-major, separate re/im */
void orc_real_basis_change(int l, double* re, double* im);
/* returns nnz (>=0) or -status; entries sorted as the reference emits them */
int orc_cg_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* v, int cap);
int orc_gaunt_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* v, int cap);
int orc_wigner_d(int l, const double* R9, double* D);
/* rotate a flat vector of single copies with degrees ls[0..n) */
int orc_rotate(const int* ls, int n, const double* x, const double* R9, double* out);

/* ---- sphere (proj/src/sphere.cpp) ---- */
int orc_gauss_legendre(int n, double* nodes, double* weights);
/* rows (lmax+1)(lmax+2)/2, cols n: lam[row*n + j] */
int orc_legendre_lambda(int lmax, const double* cos_theta, int n, double* lam);
/* synthesis on make_grid(Lgrid): out [n_theta][n_phi] */
int orc_to_sphere(const int* ls, int n, const double* x, int Lgrid, double* F, uint64_t* ops);
int orc_from_sphere_select(int Lgrid, const double* F, const int* degrees, int nd, double* out,
                           uint64_t* ops);

/* ---- CGTP (proj/src/cgtp.cpp) ---- impl: 0 naive, 1 sparse */
int orc_num_paths(int L1, int L2, int L3);
int orc_valid_paths(int L1, int L2, int L3, int* l1, int* l2, int* l3, int cap);
int orc_cgtp_path(int impl, int l1, int l2, int l3, const double* x, int nx, const double* y,
                  int ny, double* out, int nout, uint64_t* ops);
/* returns output dim (>=0) or -status; out may be NULL to query the dim */
int orc_cgtp_mimo(int impl, const int* xls, int nx, const double* x, const int* yls, int ny,
                  const double* y, double* out, uint64_t* ops);

/* ---- GTP (proj/src/gtp.cpp) ---- */
int orc_gtp_grid_select(const int* xls, int nx, const double* x, const int* yls, int ny,
                        const double* y, const int* degrees, int nd, double* out, uint64_t* ops);
int orc_gtp_fourier_select(const int* xls, int nx, const double* x, const int* yls, int ny,
                           const double* y, const int* degrees, int nd, double* out,
                           uint64_t* ops);
int orc_weighted_gtp(const int* xls, int nx, const double* x, const int* yls, int ny,
                     const double* y, const double* a, int na, const double* b, int nb,
                     const double* c, int nc, int L3, double* out, uint64_t* ops);
/* Fourier tables for input band L: which=0 encode (l<=L), 1 decode (l<=2L).
 * Flattened per (l,m) in l*l+(m+l) order: counts[(lmax+1)^2], then entries
 * (u, v, re, im).  Returns total entries or -status. */
int orc_fourier_tables(int L, int which, int* counts, int* u, int* v, double* re, double* im,
                       int cap);

/* ---- MTP (proj/src/mtp.cpp) ---- impl: 0 naive, 1 sparse */
int orc_mtp_l_tilde(int L1, int L2, int L3);
int orc_mtp_embed(const int* ls, int n, const double* x, int lt, int impl, double* X,
                  uint64_t* ops);
int orc_mtp_matmul(int dt, const double* X, const double* Y, double* Z, uint64_t* ops);
int orc_mtp_extract_select(int dt, const double* Z, const int* degrees, int nd, int lt, int impl,
                           double* out, uint64_t* ops);
int orc_mtp(const int* xls, int nx, const double* x, const int* yls, int ny, const double* y,
            int L3, int impl, int lt_override, double* out, uint64_t* ops);
double orc_mtp_path_weight(int l1, int l2, int l3, int lt);

/* ---- bench (proj/src/bench.cpp) ----
 * kind: 0 cgtp, 1 gtp, 2 mtp ; impl: 0 naive, 1 sparse, 2 grid, 3 fourier ;
 * mode: 0 siso, 1 simo, 2 mimo */
int64_t orc_count_ops(int kind, int impl, int mode, int L);
long orc_expressivity_count(int kind, int L);
/* MIMO output dim for kind at band L (cgtp (L+1)^4, else (2L+1)^2) */
int orc_mimo_out_dim(int kind, int L);
/* Batched MIMO application (run_once semantics, L3 = 2L) over B samples x C
 * channels; x [B][C][Din], y [B][Din] if y_shared else [B][C][Din],
 * out [B][C][Dout].  Batch-parallel over nthreads std::threads. */
int orc_batch_mimo(int kind, int impl, int L, int64_t B, int C, int y_shared, const double* x,
                   const double* y, double* out, int nthreads);
/* same, fp32 in/out (inputs promoted to fp64, outputs rounded) */
int orc_batch_mimo_f32(int kind, int impl, int L, int64_t B, int C, int y_shared, const float* x,
                       const float* y, float* out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
