/*
 * tpo_capi.h -- C ABI of the B200-native TPO hot path (libtpo_b200.so).
 *
 * Drop-in boundary for the reference so3tpo operator API
 * (/root/reference/proj/include/tpo/{cgtp,gtp,mtp}.hpp).  The reference has
 * one-TP-per-call, fp64, Eigen-typed entry points and no FFI for the hot path
 * (its only binding is pybind11, proj/bindings/py_core.cpp:74-109); the
 * entry points below are what that binding (and the C++ API in
 * include/tpo/*.hpp) calls instead.  Plain pointers and sizes only.
 *
 * Data layout: every irreps vector is a single-copy
 * tower 0..L, flat, degree-major, m = -l..l inside a degree
 * (proj/include/tpo/irreps.hpp:61-62).  Batched tensors are row-major
 *   x   [batch][channels][(L1+1)^2]            fp32
 *   y   [batch][(L2+1)^2]   if y_shared         fp32
 *       [batch][channels][(L2+1)^2] otherwise
 *   out [batch][channels][tpo_out_dim(kind, L1, L2, L3)]   fp32
 * Device-pointer entry points are asynchronous on `stream` (a cudaStream_t,
 * NULL = legacy default stream).  Host-pointer entry points (`_host`) copy
 * in, launch, copy out and synchronize.
 *
 * Errors: every call returns TPO_OK (0) or a positive status; the message is
 * in tpo_last_error() (thread-local).  Status mirrors the reference's
 * exceptions: TPO_EINVAL <-> std::invalid_argument (e.g.
 * proj/src/cgtp.cpp:75,148-150, proj/src/gtp.cpp:198,209-210,
 * proj/src/mtp.cpp:49-51,104-105), TPO_ERANGE <-> std::out_of_range
 * (proj/src/irreps.cpp:65-68), TPO_ERUNTIME <-> runtime_error/logic_error
 * (table self-checks, proj/src/gtp.cpp:105-106,137-138,175-177),
 * TPO_ECUDA for CUDA failures (no reference analogue).
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with TPO_ECUDA.
 */
#ifndef TPO_CAPI_H
#define TPO_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPO_OK 0
#define TPO_EINVAL 1
#define TPO_ERANGE 2
#define TPO_ERUNTIME 3
#define TPO_ECUDA 4

/* product kinds (proj/include/tpo/bench.hpp:12 BenchImpl x expressivity.hpp Kind) */
#define TPO_KIND_CGTP 0        /* cgtp_mimo, path-sparse     proj/src/cgtp.cpp:145-177 */
#define TPO_KIND_GTP_GRID 1    /* gtp_grid / grid_select     proj/src/gtp.cpp:197-260 */
#define TPO_KIND_GTP_FOURIER 2 /* gtp_fourier                proj/src/gtp.cpp:217-327 */
#define TPO_KIND_MTP 3         /* mtp                        proj/src/mtp.cpp:99-117   */

typedef struct tpo_ctx tpo_ctx;

/* Library / context ------------------------------------------------------ */
const char* tpo_last_error(void);
const char* tpo_version(void);
/* Creates a context bound to CUDA device `device`; device tables (CG term
 * lists, quadrature/GEMM operands, Fourier tables) are built lazily per
 * (kind, L1, L2, L3) and cached for the context lifetime, like the
 * reference's process-lifetime memo caches (proj/src/wigner.cpp:64-81). */
int tpo_ctx_create(int device, tpo_ctx** out);
int tpo_ctx_destroy(tpo_ctx* ctx);
/* Number of kernel launches issued through this context so far. */
int64_t tpo_ctx_launches(const tpo_ctx* ctx);

/* Shapes ------------------------------------------------------------------ */
/* (L+1)^2 */
int64_t tpo_tower_dim(int L);
/* cgtp: sum over valid paths of (2 l3 + 1)  (= (L1+1)^2 (L2+1)^2), L3 ignored;
 * gtp_grid / gtp_fourier / mtp: (L3+1)^2.  Negative status on bad args. */
int64_t tpo_out_dim(int kind, int L1, int L2, int L3);
/* MTP carrier degree ceil(max(L1,L2,L3)/2), proj/src/mtp.cpp:94-97 */
int tpo_mtp_l_tilde(int L1, int L2, int L3);

/* Batched device-pointer entry points ------------------------------------ */
/* replaces tpo::cgtp_mimo(x, y, CgtpImpl::sparse) -- proj/include/tpo/cgtp.hpp:52-54 */
int tpo_cgtp_mimo_f32(tpo_ctx* ctx, int L1, int L2, const float* x, const float* y, float* out,
                      int64_t batch, int64_t channels, int y_shared, void* stream);
/* replaces tpo::gtp_grid(x, y, L3) -- proj/include/tpo/gtp.hpp:15-16 */
int tpo_gtp_grid_f32(tpo_ctx* ctx, int L1, int L2, int L3, const float* x, const float* y,
                     float* out, int64_t batch, int64_t channels, int y_shared, void* stream);
/* replaces tpo::gtp_fourier(x, y, L3) -- proj/include/tpo/gtp.hpp:80-81 */
int tpo_gtp_fourier_f32(tpo_ctx* ctx, int L1, int L2, int L3, const float* x, const float* y,
                        float* out, int64_t batch, int64_t channels, int y_shared, void* stream);
/* replaces tpo::mtp(x, y, L3, MtpImpl::sparse, nullptr, l_tilde_override)
 * -- proj/include/tpo/mtp.hpp:41-43 ; l_tilde < 0 picks the minimal carrier */
int tpo_mtp_f32(tpo_ctx* ctx, int L1, int L2, int L3, int l_tilde, const float* x,
                const float* y, float* out, int64_t batch, int64_t channels, int y_shared,
                void* stream);
/* replaces tpo::weighted_gtp(x, y, a, b, c, L3) -- proj/include/tpo/gtp.hpp:21-24 ;
 * a[L1+1], b[L2+1], c[L3+1] are HOST arrays of per-degree weights */
int tpo_weighted_gtp_f32(tpo_ctx* ctx, int L1, int L2, int L3, const double* a,
                         const double* b, const double* c, const float* x, const float* y,
                         float* out, int64_t batch, int64_t channels, int y_shared, void* stream);

/* Backward (vector-Jacobian products) of any kind: given grad_out
 * [batch][channels][Dout], writes grad_x [batch][channels][(L1+1)^2] and
 * grad_y [batch][channels][(L2+1)^2] (either may be NULL to skip it).  The
 * reference has no backward (its paper benchmarks one);
 * this is SURVEY.md 8(f) f4.  GTP kinds reuse the forward kernels through the
 * symmetry of the real Gaunt coefficients, MTP through embed/extract adjoints
 * (same l_tilde as the forward), CGTP through transposed CG term lists.
 * y_shared != 0 is supported for grad_x only (grad_y must be NULL). */
int tpo_backward_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde, const float* x,
                     const float* y, const float* grad_out, float* grad_x, float* grad_y,
                     int64_t batch, int64_t channels, int y_shared, void* stream);

/* Generic dispatch by kind (l_tilde only used by MTP). */
int tpo_run_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde, const float* x,
                const float* y, float* out, int64_t batch, int64_t channels, int y_shared,
                void* stream);
/* Same with HOST buffers, synchronous like the reference's call: the batch is
 * cut into ~8 MiB chunks that flow through copy-in, compute and copy-out
 * streams over three device buffer sets owned by the context, so both PCIe
 * directions overlap the kernels (pinned host memory gives full overlap). */
int tpo_run_host_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde,
                     const float* x_host, const float* y_host, float* out_host, int64_t batch,
                     int64_t channels, int y_shared);

/* Several independent host-buffer requests in one call (serving-style batching of
 * heterogeneous products): their chunks flow back to back through the same copy-in /
 * compute / copy-out pipeline, so the pipeline does not drain between requests.
 * Synchronous; equivalent to n calls of tpo_run_host_f32 (same results). */
typedef struct tpo_host_request {
  int kind, L1, L2, L3, l_tilde, y_shared;
  int64_t batch, channels;
  const float* x;
  const float* y;
  float* out;
} tpo_host_request;
int tpo_run_host_batch_f32(tpo_ctx* ctx, const tpo_host_request* reqs, int n);

/* Table introspection ------------------------------------------------------
 * Real-basis CG table of (l1,l2)->l3 as the device kernels use it (mirrors
 * tpo::cg_real, proj/include/tpo/wigner.hpp:59-64, and the pybind
 * cg_table, proj/bindings/py_core.cpp:62-72).  With m1 == NULL returns the
 * entry count; otherwise fills up to `cap` entries and returns the count.
 * Negative status on error. */
int tpo_cg_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* value, int cap);
/* Torus Fourier tables of band L (tpo::fourier_tables, proj/include/tpo/gtp.hpp:76):
 * which = 0 encode (l <= L), 1 decode (l <= 2L).  counts[(lmax+1)^2] per (l,m)
 * in l*l+m+l order, entries (u, v, re, im) concatenated.  Returns the total
 * entry count (or a negative status). */
int tpo_fourier_table(int L, int which, int* counts, int* u, int* v, double* re, double* im, int cap);

/* Stage entry points ------------------------------------------------------
 * The reference's pipelines are exported stage by stage (its timing harness,
 * proj/src/bench.cpp:58-72, and its round-trip suite, proj/src/verify.cpp:256-309,
 * call the stages directly).  Batched over rows, device pointers, async on
 * `stream`; inputs are single-copy towers 0..L (sum repeated degrees first:
 * every stage is linear per entry).  Grids are make_grid(grid_L): n_theta =
 * grid_L + 1 Gauss-Legendre rows (ascending cos theta) x n_phi = 2 grid_L + 1
 * uniform columns, F row-major [n_theta][n_phi] per row. */
/* replaces tpo::to_sphere(x, make_grid(grid_L)) -- proj/include/tpo/sphere.hpp:73-74 ;
 * x [batch][(L+1)^2] -> F [batch][n_theta * n_phi]; EINVAL if L > grid_L */
int tpo_to_sphere_f32(tpo_ctx* ctx, int L, int grid_L, const float* x, float* F, int64_t batch, void* stream);
/* replaces tpo::detail::from_sphere_select(f, degrees) -- proj/include/tpo/sphere.hpp:86-88 ;
 * `degrees` is a HOST array; out [batch][sum (2l+1)] in the given order */
int tpo_from_sphere_f32(tpo_ctx* ctx, int grid_L, const int* degrees, int n_degrees, const float* F, float* out,
                        int64_t batch, void* stream);
/* replaces tpo::pointwise_mul -- proj/include/tpo/sphere.hpp:82-83 ; n floats */
int tpo_pointwise_mul_f32(tpo_ctx* ctx, const float* a, const float* b, float* out, int64_t n, void* stream);
/* replaces tpo::mtp_embed(x, l_tilde) -- proj/include/tpo/mtp.hpp:20-22 ;
 * x [batch][(L+1)^2] -> X [batch][dt][dt] row-major, dt = 2 l_tilde + 1; EINVAL if L > 2 l_tilde */
int tpo_mtp_embed_f32(tpo_ctx* ctx, int L, int l_tilde, const float* x, float* X, int64_t batch, void* stream);
/* replaces tpo::mtp_matmul(X, Y) -- proj/include/tpo/mtp.hpp:36-37 ; Z[b] = X[b] Y[b], dt x dt */
int tpo_mtp_matmul_f32(tpo_ctx* ctx, int dt, const float* X, const float* Y, float* Z, int64_t batch, void* stream);
/* replaces tpo::mtp_extract_select(Z, degrees, l_tilde) -- proj/include/tpo/mtp.hpp:30-33
 * (mtp_extract = degrees 0..L3); degrees past 2 l_tilde give zero blocks; `degrees` is a HOST array */
int tpo_mtp_extract_f32(tpo_ctx* ctx, int l_tilde, const int* degrees, int n_degrees, const float* Z, float* out,
                        int64_t batch, void* stream);
/* replaces tpo::apply_linear(LinearLayer(in, out), x) -- proj/include/tpo/irreps.hpp:77-107 ;
 * irreps as (mul, l) lists (HOST), one weight per (input copy, output copy) of equal degree in the
 * reference's connection order (proj/src/irreps.cpp:95-104); x [batch][dim in] -> out [batch][dim out] */
int tpo_apply_linear_f32(tpo_ctx* ctx, const int* in_mul, const int* in_l, int n_in, const int* out_mul,
                         const int* out_l, int n_out, const double* weights, int n_weights, const float* x, float* out,
                         int64_t batch, void* stream);
/* replaces tpo::wigner_d(l, rot) for l = 0..L -- proj/include/tpo/wigner.hpp:86 ; R [n][9] row-major
 * rotation matrices (device, fp64) -> D [n][tpo_wigner_d_size(L)] (device, fp64): the blocks D^0..D^L,
 * each (2l+1) x (2l+1) row-major, by the reference's recursion */
int tpo_wigner_d_f64(tpo_ctx* ctx, int L, const double* R, double* D, int64_t n, void* stream);
int64_t tpo_wigner_d_size(int L);
/* replaces tpo::rotate(x, rot) -- proj/include/tpo/wigner.hpp:89 ; x [batch][channels][(L+1)^2];
 * n_rot rotations R [n_rot][9] (device, fp64): sample b uses rotation b * n_rot / batch (1 = shared,
 * batch = one per sample) */
int tpo_rotate_f32(tpo_ctx* ctx, int L, const double* R, int64_t n_rot, const float* x, float* out, int64_t batch,
                   int64_t channels, void* stream);

/* Per-path weighted CGTP (the MACE "uvu" edge product): path p = (l1, l2, l3) in
 * the reference's order (proj/src/cgtp.cpp:152-163) is scaled by w[e * n_paths + p] for edge e =
 * row / channels (w_per_edge != 0; the usual case, weights from a radial network per edge) or by
 * w[p] for every row (w_per_edge == 0); w is a DEVICE fp32 array.  Fused into the shared-y edge
 * kernel's M_y (config C4 shape), an output scaling pass otherwise. */
int tpo_cgtp_num_paths(int L1, int L2);
int tpo_cgtp_weighted_f32(tpo_ctx* ctx, int L1, int L2, const float* w, int w_per_edge, const float* x,
                          const float* y, float* out, int64_t batch, int64_t channels, int y_shared,
                          void* stream);

/* Host tables / analysis (table-time, no device) ----------------------------
 * gaunt_real (proj/include/tpo/wigner.hpp:64, pybind cg_table(gaunt=True)): same contract as
 * tpo_cg_real. */
int tpo_gaunt_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* value, int cap);
/* make_grid(L) nodes / weights: L+1 ascending cos(theta) and Gauss-Legendre weights (sum 2)
 * (proj/include/tpo/sphere.hpp:49-55) ; either pointer may be NULL */
int tpo_s2_grid(int L, double* cos_theta, double* weights);
/* legendre_lambda_table (proj/include/tpo/sphere.hpp:33): lam[idx(l,m) * n + j], idx = l(l+1)/2 + m */
int tpo_legendre_lambda(int lmax, const double* cos_theta, int n, double* lam);
/* mtp_path_weights (proj/include/tpo/mtp.hpp:48); NaN on error */
double tpo_mtp_path_weight(int l1, int l2, int l3, int l_tilde);
/* count_ops (proj/include/tpo/bench.hpp:45): the reference's instrumented multiply count of one
 * application; kind 0 cgtp / 1 gtp / 2 mtp, impl 0 naive / 1 sparse / 2 grid / 3 fourier,
 * mode 0 siso / 1 simo / 2 mimo.  Negative status on error. */
int64_t tpo_count_muls(int kind, int impl, int mode, int L);

/* Kernel selection for the two Gaunt products (for tests/bench): 0 auto,
 * 1 force the tcgen05 kernels (fused, or degree groups up to L = 14; fails
 * past that), 2 force the SIMT kernels (separable grid GTP; direct half-plane
 * spectral convolution for the Fourier GTP), 3 force the separable row-quad
 * kernel (grid: as 2; Fourier: the reference torus folded to theta in [0, pi]).
 * Returns the previous setting. */
int tpo_set_gtp_grid_path(tpo_ctx* ctx, int path);
/* Accumulation precision of the tcgen05 Gaunt products (grid / Fourier).  The tensor pipe rounds
 * its fp32 accumulator toward zero once per MMA, so long accumulation chains are cut into segments
 * summed in fp32.  0 (default): segments past the per-operator limits, normwise
 * error <= 6.8e-6 on adversarial rows at every L; 1 (strict): segments past 20 K-steps for every
 * shape, <= ~4e-6, about 25% slower at L = 8..10.  Returns the previous mode. */
int tpo_set_precision(tpo_ctx* ctx, int mode);
/* Which kernel the last GTP-grid / GTP-Fourier call used (1 tc, 2 simt, 3 small-degree SIMT,
 * 4 separable torus kernel for the Fourier GTP). */
int tpo_last_gtp_grid_path(const tpo_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
