/*
 * mpid.h — C ABI of the B200-native mixed-precision interpolative decomposition
 * (ID) hot path, after arXiv 2012.00706 ("PAPER.md"; P:L = PAPER.md line L).
 *
 * The operation (Algorithm 2; Eq. (4)-(8)):
 *   given A_D (m x n, fp64), a target rank k (or a tolerance eps), a low-
 *   precision format and a range scaling,
 *     1. A_L = fl_L(s * A_D)                                  (Alg. 2 line 2)
 *     2. A_L Z = Q R, rank-k column-pivoted Householder QR in the simulated
 *        low precision (fp16/fp32 storage, fp32 arithmetic)   (Alg. 2 line 4, Eq. (6)-(7))
 *     3. I = Z(:, 1:k); P(:, I) = I_k, P(:, J) = T with
 *        T = R11^{-1} R12 (R mode, Eq. (8)) or the fp64 least-squares fit of
 *        A_D(:, J) on A_D(:, I) (LSQ mode)             (Alg. 2 lines 5-7)
 *     4. ||A_D - A_D(:, I) P||_F evaluated in fp64             (Remark 2)
 *
 * Conventions
 *   - All matrices are column-major.  Indices are 0-based.
 *   - Every call is collective over the `nranks` ranks of a row-sharded matrix:
 *     rank r owns rows [row_offset, row_offset + m_local) of A_D.  With
 *     nranks > 1 the per-step reductions use the caller's NCCL communicator
 *     (an ncclComm_t passed as void*; see id_nccl_* below).  Results are
 *     identical on all ranks.
 *   - Errors: no C++ exception crosses the ABI; each call returns an id_status
 *     and id_last_error() gives a message.  ID_ERR_CUDA / ID_ERR_NCCL leave the
 *     handle unusable (destroy it).
 *   - Ownership: A_D is borrowed (read-only, must outlive the handle); the
 *     workspace is caller-owned device memory of id_workspace_bytes() bytes
 *     (e.g. a torch uint8 tensor); outputs go to caller memory as stated per
 *     call.  All work is enqueued on the caller's CUDA stream; calls that
 *     return host values synchronise that stream.
 */
#ifndef MPID_H
#define MPID_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpid_ctx* id_handle;

/* Low-precision storage formats, Table 1.  Arithmetic is fp32 in both
 * ("simulated half").  ID_FP64 is the paper's double ID (Algorithm 1,
 * P:143-155; Â_D of P:196): fp64 storage and arithmetic, every product-then-add
 * rounded twice (DMUL, DADD; reading R16); it needs a workspace sized
 * with fmt = ID_FP64, the FFMA formation, and nb <= 8. */
typedef enum { ID_FP16 = 1, ID_FP32 = 2, ID_FP64 = 3 } id_format;

/* Range scaling before rounding (BASELINE.json configs[1]; reading R7):
 * NONE: s = 1; MAXABS: s = 1/max|a_ij|; POW2: s = 2^-ceil(log2 max|a_ij|). */
typedef enum { ID_SCALE_NONE = 0, ID_SCALE_MAXABS = 1, ID_SCALE_POW2 = 2 } id_scaling;

/* Coefficient modes: R = T from the low-precision R (Eq. (8), Alg. 2 line 5);
 * LSQ = fp64 least-squares refit against A_D(:, I). */
typedef enum { ID_COEF_R = 0, ID_COEF_LSQ = 1 } id_coef_mode;

typedef enum {
  ID_OK = 0,
  ID_ERR_ARG = 1,        /* null pointer / invalid enum / bad leading dimension */
  ID_ERR_DIM = 2,        /* k out of range, shard geometry inconsistent, workspace too small */
  ID_ERR_OVERFLOW = 3,   /* A_L has an Inf after scaling and rounding, or A_D
                            holds a NaN / Inf */
  ID_ERR_UNDERFLOW = 4,  /* selected pivot norm^2 below the normal range of the working
                            precision (fp32; fp64 for ID_FP64 and the sketch), or, for Gram
                            pivoting, a non-positive residual diagonal; k_out holds
                            the completed steps, piv_out[0:k_out] valid */
  ID_ERR_DEGENERATE = 5, /* R11 or the skeleton Gram matrix is numerically singular */
  ID_ERR_DOMAIN = 6,     /* eps outside [0, 1) */
  ID_ERR_CUDA = 7,
  ID_ERR_NCCL = 8,
  ID_ERR_OOM = 9,
  ID_ERR_STATE = 10      /* called out of order (create -> qrcp -> coeffs -> error) */
} id_status;

/* Numerical-model knobs of the QRCP (readings R4-R6).  NULL = defaults. */
typedef struct {
  int32_t nb;        /* store interval = panel width: the trailing matrix is re-stored
                        in the low format every nb steps (1 = SPEC's store-after-every-
                        update); 0 = default (4 with the FFMA formation, 16 otherwise).
                        1 <= nb <= 32 (<= 16 with FFMA formation). */
  int32_t use_graph; /* 0 or 1 (default) = capture the k-step loop in a CUDA graph
                        and replay it; -1 = plain stream launches. */
  int32_t profile_pass; /* 1 = bracket every panel-pass launch with CUDA events
                           (id_stats.t_pass_ms); adds event nodes between kernels. */
  int32_t formation; /* how the pending update A~ = S - V F^T is formed each step:
                        1 = CUDA-core FFMA in step order (fp16 / fp32 / fp64 storage),
                        2 = tcgen05 tensor cores: S^T I + (-F) V^T with hi / lo fp16
                        operands accumulated in TMEM (fp16 storage with range scaling,
                        n <= 2048; R14).
                        3 = Gram pivoting (the paper's "sketching"
                        future work P:402; R17): no k-step panel passes;
                        G = A_L^T A_L on tcgen05 (kind::f16, fp32 accumulation drained
                        into fp64 every 2048 rows), then a pivoted Cholesky of G in
                        fp64 gives the pivots and R (fp16 only; nb ignored).  Squares
                        the condition number: pivots agree with the Householder QRCP
                        while the residual norms stay above ~sqrt(2048 u32) max||a||.
                        4 = sketched pivoting (NEXT-4, second option; R18):
                        Y = Omega A_L with a Rademacher Omega of l >= k_max + 10 rows
                        (see sketch_oversample; seed = sketch_seed) on tcgen05,
                        then an fp64 Householder QRCP of Y; fp16 only; needs
                        l rounded up to 128 <= n.  R is the sketch's R factor.
                        5 = the whole QRCP in ONE launch in one SM's shared memory (fp16 /
                        fp32, a single shard with m x n x 4 B <= ~220 KB, e.g. C1), in the
                        oracle's paper model (per-operation RNE update, fp64 row-order
                        sums) bit for bit.
                        6 = the whole QRCP in ONE cooperative launch with the matrix held in
                        the shared memory of all SMs (fp16 / fp32, a single shard with m x n x 4 B
                        <= ~32 MB, e.g. C2): the same paper model, with each column's fp64 sums
                        formed per row slab and the slab partials added by a fixed warp tree
                        (opt-in: on C2 it is slower than the captured multi-kernel step).
                        Default: 5 when it applies, else 2 for fp16 with range scaling,
                        n <= 2048 and >= 16384 rows per shard, else 1. */
  int32_t sketch_oversample; /* formation 4: l = k_max + sketch_oversample; 0 = fill the
                                128-row MMA tile that k_max + 10 needs (l = 128 for k = 100) */
  int32_t sketch_seed;       /* formation 4: seed of the Rademacher sketch */
  int32_t reserved[2];
} id_qrcp_opts;

/* Per-call statistics (device-event times of the last calls, in ms). */
typedef struct {
  double scale;          /* s applied before rounding */
  double normAL_fro;     /* ||A_L||_F (global) */
  double normAD_fro;     /* ||A_D||_F (global) */
  double resid_est;      /* sqrt(sum of remaining downdated column norms^2) of A_L after k_out steps */
  double t_round_ms;     /* scale + round + initial norms */
  double t_qrcp_ms;      /* the k-step pivoted QR loop */
  double t_coef_ms;      /* id_coeffs_fp64 */
  double t_err_ms;       /* id_error */
  double t_pass_ms;      /* sum of the panel-pass kernel times (dominant kernel), when profiled */
  int64_t pass_launches; /* number of panel-pass launches in the last QRCP */
  int64_t kernel_launches; /* kernels launched by the last qrcp+coeffs+error sequence */
  int32_t k_out;
  int32_t nb;
  int32_t status_qrcp;
  int32_t formation;     /* formation used by the last QRCP (see id_qrcp_opts) */
  int32_t lsq_path;      /* last id_coeffs_fp64: 0 R mode, 1 LSQ preconditioned by the QRCP's R11
                            (one Cholesky QR pass), 2 LSQ by CholeskyQR2 (fallback) */
  int32_t fp64_engine;     /* engine of the last id_coeffs_fp64's LSQ GEMMs (W, G2): 1 DMMA, 2 int8
                              tensor cores (Ozaki scheme; id_set_fp64_engine); 0 for R mode */
  int32_t fp64_engine_err; /* engine of the last id_error's fused GEMM (1 DMMA, 2 int8 Ozaki) */
  int32_t reserved[1];
  double t_host_launch_ms; /* host time of the QRCP graph launch call */
  double t_call_gpu_ms;    /* device time of the whole id_qrcp_lowprec call on the caller's stream */
} id_stats;

/* Bytes of device workspace for a shard of m_local rows, n columns, rank <= k_max,
 * store interval nb (0 = default), storage format fmt.  host_AD = 1 reserves room
 * for a device copy of a host-resident A_D, host_AD = 2 only the staging buffers of a
 * host A_D streamed in row blocks (id_create_ex).  ID_FP16 and ID_FP32 share one layout;
 * ID_FP64 sizes the larger fp64 layout.  The handle carves its workspace for the
 * format of the current call (id_qrcp_lowprec / id_round_only); switching between a
 * low format and ID_FP64 re-carves it, which drops the cached CUDA graphs and the
 * previous results, and fails with ID_ERR_DIM if k_max no longer fits. */
size_t id_workspace_bytes(int64_t m_local, int64_t n, int32_t k_max, int32_t nb,
                          id_format fmt, int32_t host_AD);

/* Create a handle over this rank's shard of A_D.
 *   A_D        column-major m_local x n, leading dimension ld >= m_local; device
 *              memory, or host memory (pinned recommended), detected with
 *              cudaPointerGetAttributes — a host A_D is copied into the
 *              workspace on `stream` (host_AD must have been set in
 *              id_workspace_bytes).
 *   m_global   rows of the whole matrix; row_offset = first global row of the shard.
 *   workspace  caller-owned device memory, >= id_workspace_bytes(...) bytes,
 *              256-byte aligned.
 *   nccl_comm  ncclComm_t (as void*) when nranks > 1, else NULL; a communicator
 *              given with nranks == 1 is still used for every reduction.  A loopback
 *              group from id_loopback_create (nranks handles on one device) is
 *              accepted in its place.
 *   stream     cudaStream_t (as void*); NULL = legacy default stream. */
id_status id_create(id_handle* h, const double* A_D, int64_t m_global, int64_t m_local,
                    int64_t row_offset, int64_t n, int64_t ld, void* workspace,
                    size_t ws_bytes, void* nccl_comm, int32_t rank, int32_t nranks,
                    void* stream);

/* id_create with flags.  ID_CREATE_STREAM_HOST: a host A_D is streamed in row blocks
 * (SURVEY §8(b) ownership clause; needed when the shard does not fit the GPU, e.g. C5 at
 * P <= 2) instead of being copied whole: the workspace is sized with host_AD = 2 in
 * id_workspace_bytes (two staging blocks of <= 1 GiB instead of m_local x n doubles).  The
 * rounding (a max |a| pass when scaling, then the rounding pass), the LSQ product
 * W = Q1^T A_D(:, J) and the error read A_D block by block through two staging buffers,
 * the copies (on an internal stream) overlapped with the kernels of the previous block;
 * A_D(:, I) is copied column by column.  Pinned host memory is needed for the copies to
 * overlap; A_D must stay valid and unchanged for the handle's life.  With a streamed A_D
 * id_error_ex offers only (skeleton 0, norm 0), and the QRCP is not captured in a CUDA
 * graph.  Without the flag a host A_D is copied whole when the workspace holds it
 * (host_AD = 1 sizing) and streamed otherwise. */
#define ID_CREATE_STREAM_HOST 1
/* optional: stream blocks of 2^x rows (x >= 8; default ~1 GiB per block) */
#define ID_CREATE_STREAM_ROWS_LOG2(x) ((x) << 8)
id_status id_create_ex(id_handle* h, const double* A_D, int64_t m_global, int64_t m_local,
                       int64_t row_offset, int64_t n, int64_t ld, void* workspace,
                       size_t ws_bytes, void* nccl_comm, int32_t rank, int32_t nranks,
                       void* stream, int32_t flags);

/* Steps 1-2: scale, round, pivoted QR.  eps <= 0: fixed rank k_max; eps in (0,1):
 * stop at the first k with sqrt(sum_{unpivoted} ||r_i||^2) <= eps ||A_L||_F
 * (reading R8), k <= k_max.  Writes k_out (host) and
 * piv_out[0:k_out] (host, 0-based original column indices = I, in pivot order).
 * Synchronises the stream. */
id_status id_qrcp_lowprec(id_handle h, id_format fmt, id_scaling scaling, int32_t k_max,
                          double eps, const id_qrcp_opts* opts, int32_t* k_out,
                          int32_t* piv_out);

/* Step 3: P (k_out x n, column-major, leading dimension ldp >= k_out) in fp64 into
 * caller DEVICE memory P_out; P(:, I) is exactly I_k.  Requires a successful QRCP.
 * ID_COEF_R: T = R11^{-1} R12 from the QRCP's R (fp64 triangular solve).  ID_COEF_LSQ:
 * the fp64 least-squares fit of A_D(:, J) on A_D(:, I), by a Cholesky QR preconditioned
 * with the QRCP's R11, rerun as CholeskyQR2 when that preconditioner is too weak
 * (id_stats.lsq_path).  ID_ERR_DEGENERATE if A_D(:, I) is numerically rank deficient.
 * Synchronises the stream. */
id_status id_coeffs_fp64(id_handle h, id_coef_mode mode, double* P_out, int64_t ldp);

/* Step 4: ||A_D - A_D(:, I) P||_F and its ratio to ||A_D||_F (host scalars,
 * identical on all ranks), using the P of the last id_coeffs_fp64. */
id_status id_error(id_handle h, double* abs_fro, double* rel_fro);

/* Engine of the two large fp64 GEMMs of steps 3-4 (the LSQ products G2 = Q1^T Q1 and
 * W = Q1^T A_D(:, J), and the error's A_D(:, I) T).  Both compute the paper's fp64
 * quantities (Remark 2 P:199-201); they differ in how the products are evaluated:
 *   1 = fp64 tensor cores (DMMA, mma.sync m8n8k4.f64), every product and sum in fp64;
 *   2 = int8 tensor cores (tcgen05 kind::i8) by the Ozaki scheme: each operand row/column
 *       split into eight 7-bit slices under one power-of-two exponent, the 36 slice products
 *       with p + q <= 7 accumulated exactly in int32 and recombined in fp64 — per-product
 *       error < 1.3e-16 relative to 2^(Ea+Eb); needs k <= 128, a device-
 *       resident A_D (not ID_CREATE_STREAM_HOST), k < n <= 64 x SMs and the error kernel's
 *       shared memory (n - k <= ~4000 at k = 128) (else ID_ERR_ARG at the call);
 *   0 = automatic (default): 2 where it applies with >= 32768 rows per shard (faster on
 *       C4: coefficients 14.8 vs 19.6 ms, error 9.2 vs 14.1 ms), else 1.
 * Takes effect from the next id_coeffs_fp64 / id_error; id_stats reports the engine used. */
id_status id_set_fp64_engine(id_handle h, int32_t engine);

/* The paper's variants and metrics, using the P of the last
 * id_coeffs_fp64:
 *   skeleton 0 = A_D(:, I)            (mixed ID  Â_M = A_D(:, I) P)
 *            1 = fl_L(s A_D(:, I))/s  (low-precision skeleton, Â_L)
 *   norm     0 = Frobenius, exact fused fp64 reduction (as id_error)
 *            2 = spectral norm ("relative accuracy in terms of the matrix 2-norm"):
 *                power iteration x -> E^T E x on E = A_D - X P, never materialised,
 *                `iters` iterations (0 = 40) from x0 = 1/sqrt(n); ||A_D||_2 by the same
 *                iteration (cached per handle).  A lower estimate that converges from below.
 * Outputs: host scalars, identical on all ranks.  Requires id_coeffs_fp64. */
id_status id_error_ex(id_handle h, int32_t skeleton, int32_t norm, int32_t iters, double* abs_err,
                      double* rel_err);

/* R (k_out x n fp32, columns in pivoted order, R_jj >= 0, column-major, ldr >= k_out)
 * into DEVICE memory (an ID_FP64 R is rounded to fp32). */
id_status id_get_R(id_handle h, float* R_out, int64_t ldr);

/* The same R in fp64 (exact for every format) into DEVICE memory. */
id_status id_get_R_fp64(id_handle h, double* R_out, int64_t ldr);

/* Diagnostics of the Gram pivoting (formation 3): G = A_L^T A_L (n x n, fp64, column-major,
 * ldg >= n; the global G for row-sharded A) into DEVICE memory.  Valid after an
 * id_qrcp_lowprec with formation 3. */
id_status id_get_gram(id_handle h, double* G_out, int64_t ldg);

/* Diagnostics of the sketched pivoting (formation 4): Y = Omega A_L (l x n, fp64,
 * column-major, ldy >= l; the global sketch for row-sharded A) into DEVICE memory, and
 * l.  Omega(i, r) = +1 or -1 from the counter-based generator of synth.counter_sign
 * (stream 7, global row r).  Valid after an id_qrcp_lowprec with formation 4. */
id_status id_get_sketch(id_handle h, double* Y_out, int64_t ldy, int32_t* l_out);

/* The full column permutation Z (host, n entries, 0-based original indices in
 * pivoted order; perm_out[0:k_out] = I, the rest is the order R's trailing
 * columns are in). */
id_status id_get_perm(id_handle h, int32_t* perm_out);

/* A_L of this shard (m_local x n, column-major, ld >= m_local) into DEVICE memory:
 * uint16 fp16 bit patterns for ID_FP16, float for ID_FP32, double for ID_FP64.  Valid after
 * id_qrcp_lowprec with the same fmt and before any later re-store (i.e. it is
 * the rounded input only when called right after id_round_only). */
id_status id_get_AL(id_handle h, void* out, int64_t ld);

/* Step 1 alone (scale + round + norms), for bit-exact checks of A_L. */
id_status id_round_only(id_handle h, id_format fmt, id_scaling scaling);

id_status id_get_stats(id_handle h, id_stats* out);
const char* id_last_error(id_handle h);
void id_destroy(id_handle h);

/* NCCL plumbing (the library dlopen()s the libnccl.so.2 already loaded by the
 * process, e.g. PyTorch's).  The unique id is 128 bytes; broadcast it with any
 * transport (e.g. torch.distributed), then every rank calls id_nccl_comm_init. */
int32_t id_nccl_unique_id_bytes(void);
id_status id_nccl_get_unique_id(void* out);
id_status id_nccl_comm_init(void** comm, const void* unique_id, int32_t nranks, int32_t rank);
id_status id_nccl_comm_destroy(void* comm);

/* Loopback group: nranks handles of ONE process on ONE device stand in for nranks GPUs
 * (the row-sharded path of SURVEY §8(e) exercised on a single GPU; SURVEY §4 tests/dist
 * (i)).  Pass the returned pointer as nccl_comm to id_create of each rank's handle and
 * drive each handle from its own host thread: every reduction synchronises the
 * handle's stream, copies its buffer to the host, waits for all ranks (120 s timeout ->
 * ID_ERR_NCCL) and receives the slots reduced in rank order 0..nranks-1 (sum or max), so
 * every rank gets the same bits.  Handles on a loopback group never capture CUDA graphs.
 * The group is caller-owned; destroy it after its handles.  id_loopback_calls returns
 * the number of completed collectives (-1 for a pointer that is not a loopback group). */
id_status id_loopback_create(void** comm, int32_t nranks);
int64_t id_loopback_calls(void* comm);
void id_loopback_destroy(void* comm);

/* Library version and build target. */
const char* id_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MPID_H */
