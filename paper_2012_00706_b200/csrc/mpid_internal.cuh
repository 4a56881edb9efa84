// Internal definitions shared by the CUDA translation units of libmpid.so.
// Not part of the ABI (include/mpid.h is).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <algorithm>

namespace mpid {

// ---------------------------------------------------------------------------
// Data layout of the stored low-precision matrix S (A_L, re-stored every nb
// steps): "8-row interleaved column-major".  Element (r, c) of the m_pad x n
// shard lives at index ((r >> 3) * n + c) * 8 + (r & 7).  One 8-row group of
// one column is 16 bytes (fp16) or 32 bytes (fp32) and a row group of all n
// columns is contiguous, so a warp whose lanes take 32 consecutive columns of
// one row group reads 512 B (fp16) / 1 KB (fp32) contiguous bytes.
// ---------------------------------------------------------------------------
constexpr int RG = 8;                  // rows per group
constexpr int NB_MAX = 32;             // max store interval (pending reflectors; 16 for the FFMA pass)
constexpr int NSLOT = NB_MAX + 1;      // cyclic slots for u / f vectors
constexpr int PASS_THREADS = 256;      // 8 warps
constexpr int PASS_WARPS = PASS_THREADS / 32;
constexpr int PASS_TILE_G = 32;        // row groups per tile (256 rows)
constexpr int MAX_RED_BLOCKS = 1024;   // max partial-sum rows per step

struct DevScalars {                   // device-resident per-call state
  double scale;        // s
  double maxabs;       // max |a_ij| (global)
  double normAD2;      // ||A_D||_F^2 (global)
  double normAL2;      // ||A_L||_F^2 (global)
  double eps2normAL2;  // (eps ||A_L||_F)^2, 0 = fixed rank
  double resid2;       // remaining norm mass after the last completed step
  int32_t overflow;    // any Inf in A_L
  int32_t done;        // QRCP finished early (tolerance / underflow)
  int32_t status;      // 0 ok, ID_ERR_UNDERFLOW ...
  int32_t k_out;       // completed steps
  int32_t pivot;       // pivot chosen for the next step (current column position)
  int32_t pad[3];
};

struct PassParams {
  void* S;                 // T* stored matrix (interleaved layout)
  int64_t ngroups;         // m_pad / 8
  int64_t g_lo;            // first 8-row group holding rows >= j
  int64_t row_offset;      // global index of local row 0 (multiple of 8)
  int64_t m_local;         // real rows in this shard
  int64_t m_pad;
  int n;
  int j;                   // step (global row/col index of the pivot position)
  int j0;                  // first pending step
  int npend;               // j - j0 pending reflectors
  int store;               // write back fl(A~) after forming
  int chunks_per_split;    // 32-column chunks per blockIdx.y (set by the launcher)
  int ncols_slot;          // columns per CTA (set by the launcher)
  int gs;                  // row groups per pipeline stage (set by the launcher)
  int nst;                 // pipeline depth (set by the launcher)
  int gx_used;             // gridDim.x (set by the launcher)
  int cw, wr;              // consumer warps: column-warps x row-split warps (launcher)
  void* U;                 // [NSLOT][m_pad] raw u vectors (working precision: fp32, fp64 for fmt 3)
  const void* F;           // [NSLOT][n]   f vectors (current column order, working precision)
  const double* cvec;      // [k_max] c_t = 1/(u_t - beta_t) per step
  double* part;            // [gridDim.x][2][n] partial (w, s)
  double* xr;              // [n] row j of A~ (owner rank writes)
  const DevScalars* sc;
};
constexpr int PASS_SMEM_MAX = 225 * 1024;

// PTX helpers: mbarriers and bulk (TMA) copies, shared by the kernels --------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// bounded wait: a pipeline bug traps (an error the host sees) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 26)) __trap();
  }
}
// the same wait with the PTX suspend-time hint: a thread whose phase is not complete is
// suspended until it completes (or the 1 ms hint elapses) instead of re-polling shared
// memory, so waiting warps do not steal shared-memory cycles from TMA and the tensor cores
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity), "r"(1000000u)
        : "memory");
    if (done) return;
    if (spin > (1u << 16)) __trap();
  }
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0, 16 B aligned)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// host-side launchers ---------------------------------------------------------
// cudaFuncAttributeMaxDynamicSharedMemorySize of `func` raised to >= bytes on the current
// device (the attribute is per device; set once per (kernel, device), thread-safe)
cudaError_t smem_attr(const void* func, int bytes);
cudaError_t launch_maxabs(const double* A, int64_t m, int64_t n, int64_t ld, double* part,
                          int nblk, cudaStream_t st);
cudaError_t launch_maxabs_finish(const double* part, int nblk, DevScalars* sc, int scaling,
                                 cudaStream_t st);
cudaError_t launch_scale_from_max(DevScalars* sc, int scaling, cudaStream_t st);
// cmax (optional): atomicMax of each column's max |a_ij| (bit patterns; zeroed by the caller)
cudaError_t launch_round(int fmt, const double* A, int64_t m, int64_t m_pad, int64_t n, int64_t ld,
                         void* S, double* part, int gx, DevScalars* sc, cudaStream_t st,
                         unsigned long long* cmax = nullptr);
cudaError_t launch_init_pivot(const double* norms, int n, int* perm, DevScalars* sc,
                              cudaStream_t st);
cudaError_t launch_pass_tma(int fmt, PassParams p, int num_sms, int* gx_out, cudaStream_t st);
// the one-launch QRCP of a shared-memory-sized matrix (k_qrcp_smem.cu; the oracle's paper model)
size_t qrcp_smem_bytes(int64_t m, int n, int k);
cudaError_t launch_qrcp_smem(int fmt, const void* S, int64_t m, int n, int k_max, int nb, double eps, int* perm,
                             float* R, DevScalars* sc, cudaStream_t st);
// the one-launch cooperative QRCP of a matrix that fits all SMs' shared memory (k_qrcp_coop.cu;
// the paper model with slab-partial fp64 sums); rows per slab or 0 when it does not apply
int qrcp_coop_rows(int64_t m, int n, int num_sms);
cudaError_t launch_qrcp_coop(int fmt, const void* S, int64_t m, int n, int k_max, int nb, double eps, int* perm,
                             float* R, double* part, double* red, DevScalars* sc, int num_sms, cudaStream_t st);
// tcgen05 pass (fp16 storage; k_pass_tc.cu): operands, launch, tensor map of S
int tc_kchw(int nb);
size_t tc_vop_bytes(int64_t m_pad, int nb);
size_t tc_fop_bytes(int n, int nb);
cudaError_t launch_pass_tc(const PassParams& p, int nb, void* Vop, const void* Fop, const void* tmap,
                           const void* tmapc, int max_ctas, int* gx_out, cudaStream_t st);
int encode_tmap_S(void* tmap_out, void* S, int64_t ngroups, int n, int which);
cudaError_t launch_pass_reduce(const double* part, int gx, int n, int j, const double* xr,
                               int own_row, double* red, const DevScalars* sc, cudaStream_t st);
// F, R in the working precision: fp32 (fmt 1, 2) or fp64 (fmt 3)
// Fop != nullptr: also lay out the tcgen05 pass's F operand of step j + 1 (fp16 / fp32 only)
cudaError_t launch_reflector(int fmt, const double* red, int n, int j, int k_max, int nb, void* F, void* R,
                             double* beta, double* cvec, double* tau, int* perm, DevScalars* sc,
                             cudaStream_t st, void* Fop = nullptr);
// + (Fop != nullptr) the tcgen05 pass's F operand of step jn, laid out by extra blocks
cudaError_t launch_swap(int fmt, void* S, int64_t ngroups, int n, int jn, int j0, int steps_done,
                        void* F, void* R, int* perm, void* Sj, DevScalars* sc, cudaStream_t st, void* Fop = nullptr,
                        const double* cvec = nullptr, int nb = 16);
// k_pass_reduce + k_reflector in one launch (single shard; last-block ticket in *counter, zeroed once)
cudaError_t launch_reduce_reflect(int fmt, const double* part, int gx, int n, int j, const double* xr, int own_row,
                                  int k_max, int nb, void* F, void* R, double* beta, double* cvec, double* tau,
                                  int* perm, DevScalars* sc, double* red, double* cand, unsigned int* counter,
                                  cudaStream_t st);
cudaError_t launch_export_S(int fmt, const void* S, int64_t m_local, int n, void* out, int64_t ld,
                            cudaStream_t st);

// fp64 stage
cudaError_t launch_gather_cols(const double* A, int64_t m, int64_t ld, const int* perm, int k,
                               double* X, cudaStream_t st);
// C(k1 x n1) = X^T Y over m rows (split-K partials); column c of Y is ycmap[c] when given
cudaError_t launch_tsmm(const double* X, int64_t ldx, int k1, const double* Y, int64_t ldy, int n1,
                        int64_t m, double* part, int splits, cudaStream_t st, const int* ycmap = nullptr);
cudaError_t launch_sum_partials(const double* part, int splits, int64_t len, double* out,
                                cudaStream_t st);
cudaError_t launch_cholesky(double* G, int k, int* info, cudaStream_t st);
// out = max_i |R_ii| / min_i |R_ii| of an upper col-major k x k R (inf if a zero diagonal)
cudaError_t launch_diag_ratio(const double* R, int k, double* out, cudaStream_t st);
cudaError_t launch_trsm_left_upper(const double* R1, const double* R2, int k, const double* B,
                                   int64_t ldb, const int* map, int ncols, double* T, int64_t ldt,
                                   int mode, cudaStream_t st);
// R (k x n row-major, fp32 or fp64 when r64) -> fp64 col-major / exported col-major (fp32 or fp64 when o64)
cudaError_t launch_R_to_fp64(int r64, const void* R, int k, int n, double* Rd, cudaStream_t st);
cudaError_t launch_R_export(int r64, const void* R, int k, int n, void* out, int o64, int64_t ldr, cudaStream_t st);
cudaError_t launch_assemble_P(const double* T, int64_t ldt, int k, int n, const int* perm, double* P,
                              int64_t ldp, cudaStream_t st);
// error over the columns J: sum_{r, c} (A(r, cmap[c]) - sum_l X(r, l) T(l, c))^2, c < ncols
// X has leading dimension ldx (<= 0: m); pack = 0 reuses the T slabs packed by an earlier call
cudaError_t launch_error(const double* A, int64_t m, int64_t ld, int ncols, const int* cmap, const double* X,
                         int k, const double* T, int64_t ldt, double* part, int* nblk_out, cudaStream_t st,
                         double* tpack = nullptr, size_t tpack_cap = 0, int64_t ldx = -1, int pack = 1);
size_t ew_tpack_doubles(int64_t n, int64_t k);   // packed T slabs of the warp-specialised error kernel
// out(m x N) = X(m x K) B(K x N), all col-major
// cmax (optional): the column maxima of out (bit patterns) for the int8 engine; *cmax_done = 1
// when this launch produced them (the warp-specialised path), else the caller computes them
cudaError_t launch_nn_store(const double* X, int64_t m, int64_t ldx, const double* B, int64_t ldb, int K,
                            int N, double* out, int64_t ldo, cudaStream_t st, double* tpack = nullptr,
                            size_t tpack_cap = 0, unsigned long long* cmax = nullptr, int* cmax_done = nullptr);
cudaError_t launch_eye(double* I, int k, cudaStream_t st);
// host-streamed A_D (mpid_api.cu): acc[i] (+)= sum_y part[y * stride + i] for i < len, fixed order
cudaError_t launch_acc_rows(const double* part, int rows, int64_t stride, int64_t len, double* acc, int add,
                            cudaStream_t st);
// acc[slot] = max(part[0:nblk])
cudaError_t launch_max_into(const double* part, int nblk, double* acc, cudaStream_t st);
// NEXT-1 / NEXT-2 (k_norm2.cu): the low-precision skeleton and the 2-norm by power iteration
cudaError_t launch_gather_lowp(const double* A, int64_t m, int64_t ld, const int* perm, int k, int fmt,
                               const DevScalars* sc, double* X, cudaStream_t st);
cudaError_t launch_gemv_n(const double* A, int64_t m, int64_t ld, int n, const double* x, double* y, int subtract,
                          cudaStream_t st);
cudaError_t launch_gemv_t(const double* A, int64_t m, int64_t ld, int n, const double* y, double* part, int nblk,
                          cudaStream_t st);
cudaError_t launch_sum_cols(const double* part, int nblk, int n, const double* sub, double* out, cudaStream_t st);
cudaError_t launch_p_times(const double* P, int64_t ldp, int k, int n, const double* x, double* w, cudaStream_t st);
cudaError_t launch_pt_times(const double* P, int64_t ldp, int k, int n, const double* w, double* v, cudaStream_t st);
cudaError_t launch_normalize(const double* z, int n, double* x, double* est, int it, cudaStream_t st);
cudaError_t launch_ones(double* x, int n, cudaStream_t st);
cudaError_t launch_sum_scalar(const double* part, int nblk, double* out, cudaStream_t st);
// NEXT-4 (k_gram.cu): Gram-based pivoting — G = A_L^T A_L on tcgen05 (fp16 S), pivoted Cholesky
size_t gram_part_doubles(int64_t ngroups, int n, int num_sms);
int encode_tmap_gram(void* tmap_out, void* S, int64_t ngroups, int n);
cudaError_t launch_gram(const void* tmap, int64_t ngroups, int n, int num_sms, double* part, double* G,
                        const DevScalars* sc, cudaStream_t st);
// NEXT-4 second option: Omega^T (+-1 fp16, interleaved, lw columns), Y = Omega A_L (lw x n fp64),
// then the fp64 QRCP of Y on one CTA (ly = lw rows, zero rows beyond l)
cudaError_t launch_sketch(const void* tmapO, const void* tmapS, void* Om, int64_t ngroups, int n, int l, int lw,
                          int64_t m_local, int64_t row_offset, uint64_t base, int num_sms, double* part,
                          size_t part_doubles, double* Y, const DevScalars* sc, cudaStream_t st);
cudaError_t launch_small_qrcp(double* Y, int ly, int n, int k_max, double* snorm, int* perm, double* R64, float* R,
                              DevScalars* sc, cudaStream_t st);
// pivoted Cholesky of G (kept) on the working copy Gc, in panels of 32 steps + Schur updates
cudaError_t launch_pchol(const double* G, double* Gc, int n, int k_max, double* d, int* perm, double* R64, float* R,
                         DevScalars* sc, cudaStream_t st);

// fp64 GEMMs of the ID step on the int8 tensor cores by the Ozaki scheme (k_ozaki.cu; k <= 128)
size_t oz_slice_bytes(int64_t m_local);
size_t oz_tslice_bytes(int64_t n);
size_t oz_part_doubles(int num_sms);
bool oz_fits(int64_t n, int k, int num_sms);   // k <= 128, grid and shared memory of the int8 kernels
// cmaxq_ready: Q1's column maxima are already in cmaxq (launch_nn_store produced them)
cudaError_t launch_oz_tn(const double* Q1, int64_t m, int k, const double* AD, int64_t ld, const int* cmapJ, int nj,
                         const unsigned long long* cmaxd, unsigned long long* cmaxq, void* slices, double* part,
                         size_t part_cap, double* G2, double* W, int num_sms, cudaStream_t st, int cmaxq_ready = 0);
cudaError_t launch_oz_error(const double* AD, int64_t m, int64_t ld, int nj, const int* cmapJ, const double* AI,
                            int k, const double* T, int64_t ldt, void* slices, void* tslices, double* rsc,
                            double* fsc, double* part, int* nblk_out, int num_sms, cudaStream_t st);

}  // namespace mpid
