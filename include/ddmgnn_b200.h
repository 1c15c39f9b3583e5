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
#define DDMGNN_ASM_ONE 3      /* DDM-LU comparator: exact local solves (asm.py:84-113, "ddm-lu-1") */
#define DDMGNN_ASM_TWO 4      /* DDM-LU two-level (cli.py:69-70, "ddm-lu-2") */
#define DDMGNN_IC0 5          /* IC(0) comparator (sparse.py:170-227, "ic0") */
/* OR into the level of ddmgnn_pcg: flexible CG (Polak-Ribiere beta = <r, z - z_old> / rho
 * instead of the reference's rho'/rho at sparse.py:124; opt-in, not in the reference). */
#define DDMGNN_FLEXIBLE 0x100

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
/* DDM-LU comparator: allocate the device buffer for the K dense local inverses
 * A_i^-1 (row-major, k_i x k_i, subdomain i at offset off[i] doubles, off[K] total;
 * requires build) and return its device address for the caller to fill (setup
 * factorises on the GPU).  Enables levels DDMGNN_ASM_ONE / DDMGNN_ASM_TWO. */
int ddmgnn_alloc_local_inverses(ddmgnn_ctx* ctx, const int64_t* off, double** dev_out);
/* IC(0) comparator: factorise the context's matrix (zero fill on the lower pattern,
 * sparse.py:184-227; RuntimeError "IC(0) breakdown: ..." like the reference) and
 * enable level DDMGNN_IC0 (z = L^-T L^-1 r, sync-free triangular solves). */
int ddmgnn_set_ic0(ddmgnn_ctx* ctx);
/* The IC(0) factor L (CSR, lower, diagonal last per row); NULL buffers query nnz. */
int ddmgnn_export_ic0(ddmgnn_ctx* ctx, int64_t* nnz, int32_t* indptr, int32_t* indices,
                      double* data);
/* Node cap of the reference's batching (hybrid.py:49-68, default 100000).  Results
 * never depend on it; it only selects which error the reference would raise first. */
int ddmgnn_set_batch_cap(ddmgnn_ctx* ctx, int64_t cap);
/* Build the device layout of the per-subdomain graphs (requires matrix, geometry
 * and decomposition). */
int ddmgnn_build(ddmgnn_ctx* ctx);
/* out[0..13] = n, K, V, E, E_pad, k_max, slices, k_bar, d, lmax, n_chunks, n_big,
 * n_cluster (of the n_big oversized subdomains, those on the cluster path),
 * cluster_launches (cluster sizes in use: one launch each per chunk) */
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
/* Launch only the fused restriction + GNN kernel(s) on r_dev (sharded building block,
 * profiling aid).  Asynchronous; non-finite model states are recorded in the context's
 * status word (see ddmgnn_apply_status). */
int ddmgnn_launch_gnn_only(ddmgnn_ctx* ctx, const double* r_dev, void* stream);
/* Synchronise `stream` and report a non-finite model state recorded by the launches
 * since the last check with the reference's message ("non-finite latent state at
 * message-passing iteration k" / "non-finite model output in subdomain i"; local
 * subdomain indices); clears the status word. */
int ddmgnn_apply_status(ddmgnn_ctx* ctx, void* stream);
/* y = A x on device pointers. */
int ddmgnn_spmv(ddmgnn_ctx* ctx, const double* x_dev, double* y_dev, void* stream);

/* Device-resident PCG (sparse.py:76-127) with the GNN preconditioner at `level`
 * (or plain CG for DDMGNN_PRECOND_NONE).  b, u0 (may be NULL), u are host pointers
 * when device_ptrs == 0 and device pointers otherwise; history must hold
 * max_iter + 1 doubles (host; 1 when max_iter <= 0 — a negative max_iter runs no
 * iteration, like the reference).  On return *iterations, history[0..*iterations],
 * *converged are filled exactly like SolveReport (sparse.py:31-53).
 * level | DDMGNN_FLEXIBLE selects the opt-in flexible CG. */
int ddmgnn_pcg(ddmgnn_ctx* ctx, const double* b, const double* u0, double* u, double tol,
               int max_iter, int level, int device_ptrs, void* stream, int* iterations,
               double* history, int* converged);

/* PCG with a host-side preconditioner callback z = M(r) (host arrays of length n);
 * the Krylov recurrence still runs on the device.  The callback returns 0 on success. */
typedef int (*ddmgnn_host_precond_fn)(void* user, const double* r, double* z, int64_t n);
int ddmgnn_pcg_host_precond(ddmgnn_ctx* ctx, const double* b, const double* u0, double* u,
                            double tol, int max_iter, int flexible, ddmgnn_host_precond_fn fn,
                            void* user, int* iterations, double* history, int* converged);

/* ---- Sharded solve building blocks (one process per GPU) ----
 * A rank's context holds its group of subdomains over its local DOF set; the
 * host issues the collectives between these stream-ordered calls
 * (paper_2402_08296_b200/sharded.py).  All pointers are device pointers. */
/* Device buffers filled by ddmgnn_launch_gnn_only: zloc[V] = s_i * DSS output of
 * every batched node (hybrid.py:135), scale[K] = s_i (hybrid.py:105), r0r[K] =
 * (R0 r)_i (hybrid.py:117).  Any output pointer may be NULL. */
int ddmgnn_local_outputs(ddmgnn_ctx* ctx, double** zloc, double** scale, double** r0r);
/* Replace the partition-of-unity weights 1/multiplicity (decomp.py:184-190) that
 * build derived from the context's own subdomains — a shard passes the weights of
 * the global decomposition restricted to its local DOF set (length n). */
int ddmgnn_set_pou(ddmgnn_ctx* ctx, int64_t n, const double* pou);
/* dst[i] = src[idx[i]] and dst[idx[i]] = src[i], i < n (halo pack / unpack). */
int ddmgnn_gather(const double* src, const int32_t* idx, int64_t n, double* dst, void* stream);
int ddmgnn_scatter(const double* src, const int32_t* idx, int64_t n, double* dst, void* stream);
/* *out = x . y (fixed two-stage order; work holds >= 1184 doubles). */
int ddmgnn_dot(int64_t n, const double* x, const double* y, double* work, double* out,
               void* stream);
/* *out = x . (y - w) (same order as ddmgnn_dot; the flexible-CG numerator <r, z - z_old>). */
int ddmgnn_dot_diff(int64_t n, const double* x, const double* y, const double* w, double* work,
                    double* out, void* stream);
/* u += alpha p, r -= alpha q (sparse.py:112-113), *rr_out = r . r (sparse.py:114). */
int ddmgnn_axpy2(int64_t n, double alpha, const double* p, const double* q, double* u, double* r,
                 double* work, double* rr_out, void* stream);
/* p = z + beta p (sparse.py:126). */
int ddmgnn_xpby(int64_t n, const double* z, double beta, double* p, void* stream);
/* Device-side scalars of the distributed PCG: st = {rho, pq, alpha, rr, nb, tol, rz,
 * beta, iter, status, max_iter, rzo} (fp64, device).  op 0: alpha = rho / pq (status 3 if
 * pq <= 0, sparse.py:108-111); op 1: rel = sqrt(rr) / nb, hist[++iter] = rel, status
 * 1 converged / 2 max_iter / 4 non-finite (sparse.py:114-121); op 2: beta = rz / rho,
 * rho = rz (sparse.py:123-125); op 3 (flexible CG): beta = rzo / rho, rho = rz.
 * No-ops once status != 0. */
int ddmgnn_pcg_scalars(int op, double* st, double* hist, void* stream);
/* ddmgnn_axpy2 / ddmgnn_xpby with alpha / beta read from st (no-ops once status != 0). */
int ddmgnn_axpy2_dev(int64_t n, const double* st, const double* p, const double* q, double* u,
                     double* r, double* work, double* rr_out, void* stream);
int ddmgnn_xpby_dev(int64_t n, const double* z, const double* st, double* p, void* stream);
/* y = A x, A dense row-major k x k (the coarse inverse, sparse.py:163 / hybrid.py:117). */
int ddmgnn_dense_gemv(int64_t k, const double* a, const double* x, double* y, void* stream);
/* Gluing over a transpose map (hybrid.py:117,133-135): for DOF j < n,
 * z_j = [two_level] sum_t pou_j y[sub_t] + sum_{t: scale[sub_t] != 0} zloc[pos_t],
 * t in [tptr[j], tptr[j+1]) ascending subdomain; tent = int32 pairs (pos, sub). */
int ddmgnn_prolong(int64_t n, int two_level, const int32_t* tptr, const int32_t* tent,
                   const double* pou, const double* y, const double* scale, const double* zloc,
                   double* z, void* stream);

/* ---- Device-resident peer collectives (sharded solve without host barriers) ----
 * g <= DDMGNN_PEER_MAX ranks, this rank `me`; flags[h] = rank h's flag block
 * (int64[DDMGNN_PEER_FLAG_WORDS], zero-initialised, mapped into every rank with
 * CUDA IPC); chan < DDMGNN_PEER_CHANNELS names one call site.  Ordering is by
 * device-side epochs and acknowledgements, so the calls are stream-ordered and
 * graph-capturable; every rank must make the same sequence of calls per channel.
 * Host arrays: flags/dst/out/slots (g device pointers), send_off/recv_off (g + 1). */
#define DDMGNN_PEER_MAX 8
#define DDMGNN_PEER_CHANNELS 8
#define DDMGNN_PEER_FLAG_WORDS (DDMGNN_PEER_CHANNELS * 32)
/* Segment h of src[idx[send_off[h] .. send_off[h+1])] into dst[h] + dst_off[h]
 * (rank h's receive buffer), then signal h. */
int ddmgnn_peer_put(int g, int me, int chan, int64_t* const* flags, const double* src,
                    const int32_t* idx, const int64_t* send_off, double* const* dst,
                    const int64_t* dst_off, void* stream);
/* Wait until every rank h with a non-empty receive segment [recv_off[h], recv_off[h+1])
 * delivered this call's epoch; then ext[pos[i]] = recv[i] (pos may be NULL), and
 * with ack != 0 acknowledge to the senders (else call ddmgnn_peer_ack after the
 * kernel that consumes recv). */
int ddmgnn_peer_wait(int g, int me, int chan, int64_t* const* flags, const int64_t* recv_off,
                     const double* recv, const int32_t* pos, double* ext, int ack, void* stream);
int ddmgnn_peer_ack(int g, int me, int chan, int64_t* const* flags, const int64_t* recv_off,
                    void* stream);
/* out[h] (rank h's [g][k] buffer) row me = in[0..k), on every rank. */
int ddmgnn_peer_allgather(int g, int me, int chan, int64_t* const* flags, double* const* out,
                          const double* in, int64_t k, void* stream);
/* inout[0..k) = sum over ranks in rank order (k <= 16; identical bits on every
 * rank); slots[h] = rank h's [g][k] staging area of this channel. */
int ddmgnn_peer_allreduce(int g, int me, int chan, int64_t* const* flags, double* const* slots,
                          double* inout, int k, void* stream);
/* A wait that sees no peer for 30 s gives up and sets flags[me][DDMGNN_PEER_FLAG_WORDS - 1]
 * (the host checks it when it polls the solve status). */
/* Peer-visible buffers: zeroed cudaMalloc on `device`; 64-byte CUDA IPC handles;
 * ddmgnn_ipc_open maps a peer's buffer into this process (lazy peer access from
 * `device`, NVLink between the GPUs of one box). */
int ddmgnn_peer_alloc(int device, int64_t bytes, void** ptr);
int ddmgnn_peer_free(void* ptr);
int ddmgnn_ipc_get(void* ptr, unsigned char* handle);
int ddmgnn_ipc_open(int device, const unsigned char* handle, void** ptr);
int ddmgnn_ipc_close(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* DDMGNN_B200_H */
