/*
 * ddmgnn_b200 — C ABI of the B200-native DDM-GNN preconditioner and PCG solver.
 *
 * Drop-in boundary for the reference package `ddmgnn` 0.1.0 (pure Python; its
 * "plugin" interface is the preconditioner operator hook of `pcg`):
 *
 *   reference (pkg/src/ddmgnn/…)                      replaced by
 *   -----------------------------------------------   ------------------------------------
 *   build_ddm_gnn(a, coords, dec, model, cap)         ddmgnn_create + set_matrix +
 *     hybrid.py:84-97                                   set_geometry + set_decomposition +
 *                                                       set_model + set_coarse_inverse +
 *                                                       set_batch_cap + build
 *   build_local_graphs / extract_local_matrix /       ddmgnn_build (layout builder)
 *     local_graph_from_matrix  hybrid.py:36-46,
 *     asm.py:28-32, dss.py:173-186
 *   DdmGnnPreconditioner.__call__ / apply_ddm_gnn     ddmgnn_apply (device pointers) /
 *     hybrid.py:80-81, 112-136                          ddmgnn_apply_host (host pointers)
 *   pcg(a, b, precond, tol, max_iter, u0)             ddmgnn_pcg / ddmgnn_pcg_host_precond
 *     sparse.py:76-127;  cg  sparse.py:130-132
 *   Decomposition pou / r0   decomp.py:180-193,238-246  computed inside ddmgnn_build
 *   Factorization(coarse).solve  sparse.py:158-164   ddmgnn_set_coarse_inverse (dense fp64
 *                                                       inverse, applied as a device GEMV)
 *
 * Conventions: every function returns 0 on success or a status code
 *   1 = invalid argument (Python ValueError), 2 = runtime failure (RuntimeError),
 *   3 = CUDA error, 4 = API misuse;
 * ddmgnn_last_error() returns the message of the last failure on the calling
 * thread — for the reference's runtime errors the text is identical
 * ("matrix not SPD: <p, Ap> <= 0", "non-finite residual at iteration k",
 * "non-finite latent state at message-passing iteration k",
 * "non-finite model output in subdomain i", …).
 * Arrays are plain host or device pointers with explicit sizes; `stream` is a
 * cudaStream_t passed as void* (NULL = the context's own stream).  A context is
 * not thread-safe; all work is stream-ordered.  There is no CPU fallback: every
 * compute entry point runs CUDA kernels for sm_100a.
 */
#ifndef DDMGNN_B200_H
#define DDMGNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ddmgnn_ctx ddmgnn_ctx;

/* level values for apply / pcg */
#define DDMGNN_PRECOND_NONE 0 /* plain CG (sparse.py:130-132) */
#define DDMGNN_LEVEL_ONE 1    /* one-level GNN-Schwarz (restatement of hybrid.py:112-136 w/o :117) */
#define DDMGNN_LEVEL_TWO 2    /* two-level: + Nicolaides coarse correction (hybrid.py:117) */

const char* ddmgnn_last_error(void);
int ddmgnn_version(void);

int ddmgnn_create(int device, ddmgnn_ctx** out);
void ddmgnn_destroy(ddmgnn_ctx* ctx);
void* ddmgnn_stream(ddmgnn_ctx* ctx);

/* A in CSR with sorted column indices (fem.py:162-165); copied to the device. */
int ddmgnn_set_matrix(ddmgnn_ctx* ctx, int64_t n, int64_t nnz, const int64_t* indptr,
                      const int32_t* indices, const double* data);
/* Interior DOF coordinates, row-major (n, 2) (cli.py:58). */
int ddmgnn_set_geometry(ddmgnn_ctx* ctx, int64_t n, const double* coords);
/* K strictly ascending subdomain index arrays, concatenated (decomp.py:29-44). */
int ddmgnn_set_decomposition(ddmgnn_ctx* ctx, int64_t k, const int64_t* sub_ptr,
                             const int64_t* sub_idx);
/* Flat float64 weights in the reference's _param_arrays order (dss.py:93-99). */
int ddmgnn_set_model(ddmgnn_ctx* ctx, int k_bar, int d, double alpha, const double* params,
                     int64_t n_params);
/* Dense row-major inverse of R0 A R0^T (k x k), fp64 (asm.py:35-41). */
int ddmgnn_set_coarse_inverse(ddmgnn_ctx* ctx, int64_t k, const double* inverse);
/* Node cap of the reference's batching (hybrid.py:49-68, default 100000).  Results
 * never depend on it; it only selects which error the reference would raise first. */
int ddmgnn_set_batch_cap(ddmgnn_ctx* ctx, int64_t cap);
/* Build the device layout of the per-subdomain graphs (requires matrix, geometry
 * and decomposition). */
int ddmgnn_build(ddmgnn_ctx* ctx);
/* out[0..11] = n, K, V, E, E_pad, k_max, slices, k_bar, d, lmax, n_chunks, n_big */
int ddmgnn_info(ddmgnn_ctx* ctx, int64_t* out, int n_out);
/* Edges of subdomain `sub` as built on the device (for parity tests): src/dst local
 * indices and fp32 {dx, dy, |d|}.  Pass NULL buffers to query the count. */
int ddmgnn_export_local_graph(ddmgnn_ctx* ctx, int64_t sub, int64_t* n_edges, int32_t* src,
                              int32_t* dst, float* vec3);

/* z = M r on device pointers (both length n).  check != 0 synchronises and reports
 * the reference's error for non-finite model states; check == 0 is asynchronous. */
int ddmgnn_apply(ddmgnn_ctx* ctx, const double* r_dev, double* z_dev, int level, void* stream,
                 int check);
/* Same with host pointers: H2D copy, apply, D2H copy (end-to-end path). */
int ddmgnn_apply_host(ddmgnn_ctx* ctx, const double* r, double* z, int level);
/* Launch only the fused restriction + GNN kernel(s) on r_dev (profiling aid). */
int ddmgnn_launch_gnn_only(ddmgnn_ctx* ctx, const double* r_dev, void* stream);
/* y = A x on device pointers. */
int ddmgnn_spmv(ddmgnn_ctx* ctx, const double* x_dev, double* y_dev, void* stream);

/* Device-resident PCG (sparse.py:76-127) with the GNN preconditioner at `level`
 * (or plain CG for DDMGNN_PRECOND_NONE).  b, u0 (may be NULL), u are host pointers
 * when device_ptrs == 0 and device pointers otherwise; history must hold
 * max_iter + 1 doubles (host).  On return *iterations, history[0..*iterations],
 * *converged are filled exactly like SolveReport (sparse.py:31-53). */
int ddmgnn_pcg(ddmgnn_ctx* ctx, const double* b, const double* u0, double* u, double tol,
               int max_iter, int level, int device_ptrs, void* stream, int* iterations,
               double* history, int* converged);

/* PCG with a host-side preconditioner callback z = M(r) (host arrays of length n);
 * the Krylov recurrence still runs on the device.  The callback returns 0 on success. */
typedef int (*ddmgnn_host_precond_fn)(void* user, const double* r, double* z, int64_t n);
int ddmgnn_pcg_host_precond(ddmgnn_ctx* ctx, const double* b, const double* u0, double* u,
                            double tol, int max_iter, ddmgnn_host_precond_fn fn, void* user,
                            int* iterations, double* history, int* converged);

#ifdef __cplusplus
}
#endif

#endif /* DDMGNN_B200_H */
