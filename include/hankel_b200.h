/* hankel_b200.h — C ABI of the B200-native extreme-precision Hankel LDLT path.
 *
 * The reference (/root/reference/proj, hankel-eig v0.1.0) is a C++ library with
 * no C ABI, plugin registry or FFI of its own; its entry points
 * are the C++ functions of proj/include/hankel/ *.hpp.  This header is the thin
 * C layer *below* those entry points: each call is annotated with the reference
 * function it replaces.  Plain pointers and sizes only; no torch, no C++ types.
 *
 * Number format (host interchange, "SoA"): an array of `count` p-bit floats,
 * p = 32 * limbs, is three caller-owned host arrays
 *     uint32_t limbs[count * limbs]   little-endian mantissa words per value
 *     int32_t  exps [count]           binary exponent e
 *     int32_t  signs[count]           -1, 0 (value zero, limbs all 0) or +1
 * with value = sign * M * 2^(e - p), 2^(p-1) <= M < 2^p.  Every arithmetic
 * operation on the device is correctly rounded (round to nearest, ties to even).
 *
 * Status codes mirror the reference CLI's exit codes (proj/tools/hankel_cli.cpp:4,
 * 135-147) and its exception mapping:
 *     HK_OK 0, HK_ERR_RUNTIME 1 (CUDA/NCCL/internal   -> std::runtime_error)
 *     HK_ERR_PRECISION 2 (non-positive pivot          -> hankel::precision_error;
 *                         hk_bad_column() gives the column, ldlt.cpp:83-87)
 *     HK_ERR_INVALID 3  (bad sizes / arguments        -> std::invalid_argument)
 * hk_last_error() returns the message of the last failure on that context.
 *
 * Threading: one host thread per context; calls are synchronous on return and
 * not re-entrant.  Each context owns one CUDA device and one stream.
 */
#ifndef HANKEL_B200_H
#define HANKEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HK_OK 0
#define HK_ERR_RUNTIME 1
#define HK_ERR_PRECISION 2
#define HK_ERR_INVALID 3

#define HK_OP_FMS 0   /* out = RNE(c - a*b)  — submul_rounded, fixedpoint.cpp:146-154 */
#define HK_OP_MUL 1   /* out = RNE(a*b)      — operator*, fixedpoint.cpp:67-69 (exact there) */
#define HK_OP_ADD 2   /* out = RNE(a+b)      — operator+, fixedpoint.cpp:55-59 (exact there) */
#define HK_OP_RECIP 3 /* out = RNE(1/a)      — FixScalar::div's role, fixedpoint.cpp:71-84 */
#define HK_OP_CTA 16  /* or-flag: run FMS / MUL / RECIP with the CTA-cooperative kernels */

typedef struct hk_ctx hk_ctx;

/* ABI version (major*100 + minor). */
int hk_version(void);

/* Context on CUDA device `device` computing at p = 32*limbs bits.
 * Replaces the per-run precision choice `frac_bits` of MomentTable
 * (moments.hpp:38) / ComputeOptions::bits (pipeline.hpp:19). */
int hk_create(int device, int limbs, hk_ctx** out);
void hk_destroy(hk_ctx* ctx);
const char* hk_last_error(const hk_ctx* ctx);
int hk_bad_column(const hk_ctx* ctx);
int hk_limbs(const hk_ctx* ctx);

/* Change the context's precision p = 32*limbs (drops the cached buffers and
 * graphs, keeps the device streams and — for a sharded context — the NCCL
 * communicator, so auto_precision / scan (pipeline.cpp:74-122) re-run at a new
 * K on the same communicator).  A no-op when limbs is unchanged. */
int hk_set_limbs(hk_ctx* ctx, int limbs);

/* Host-side exact moments mu_0..mu_{count-1} of w(x)=exp(-x^beta) as p-bit
 * floats (moments.cpp:80-111: gamma_exact + moment; the factorial branch and —
 * for odd 2/beta — the half-integer sqrt(pi) branch, correctly rounded).
 * *exact = 1 iff every moment was representable without rounding. No GPU. */
int hk_moments(unsigned beta_num, unsigned beta_den, int count, int limbs, uint32_t* out_limbs,
               int32_t* out_exps, int32_t* out_signs, int* exact);

/* The 2n-1 moments of order n generated ON THE DEVICE into the context's moment
 * array (csrc/moments_dev.cuh): one CTA keeps the running factorial as an exact
 * integer in shared memory and writes RNE_p of every moment — gamma_exact's
 * factorial branch + moment + the integer -> working-precision conversion of
 * build_hankel (moments.cpp:83-89, 102-111, 113-129).  Bit-identical to
 * hk_moments + hk_load_moments; no host bigint, no H2D.  Even 2/beta only (odd
 * 2/beta needs sqrt(pi): host path, HK_ERR_INVALID here).  *exact as hk_moments.
 * hk_get_moments copies the context's 2n-1 moments back (tests). */
int hk_generate_moments(hk_ctx* ctx, unsigned beta_num, unsigned beta_den, int n, int* exact);
int hk_get_moments(hk_ctx* ctx, uint32_t* limbs, int32_t* exps, int32_t* signs);

/* Upload the 2n-1 moments (H2D).  Replaces MomentTable / build_hankel
 * (moments.hpp:36-58) as the input of the factorisation. */
int hk_load_moments(hk_ctx* ctx, int n, const uint32_t* limbs, const int32_t* exps, const int32_t* signs);

/* LDLT of H = (mu_{i+j}) on the device (S <- H, then n right-looking steps).
 * Replaces decompose_serial / decompose_parallel (ldlt.hpp:90, 97-99).
 * HK_ERR_PRECISION with hk_bad_column() on a non-positive pivot. */
int hk_ldlt(hk_ctx* ctx);

/* D_0..D_{n-1} (n values) and column `col` of L (n-col-1 values, rows col+1..n-1),
 * LdltFactors::D / L (ldlt.hpp:76-85). */
int hk_get_D(hk_ctx* ctx, uint32_t* limbs, int32_t* exps, int32_t* signs);
int hk_get_L_column(hk_ctx* ctx, int col, uint32_t* limbs, int32_t* exps, int32_t* signs);

/* First m columns of L^{-1}.  Replaces invert_L_partial_serial / _parallel
 * (inversion.hpp:40, 45-46).  hk_get_Linv returns n*m values row-major; entry
 * (r,c) is L^{-1}(r,c) for c < r, and 0 for c >= r (unit diagonal implicit). */
int hk_invert_L_partial(hk_ctx* ctx, int m);
/* hk_ldlt followed by hk_invert_L_partial(m) as ONE call — the pair compute()
 * runs back to back (pipeline.cpp:41-58).  Where both stages are latency-bound
 * (one GPU, small p) the row-elimination steps of L^{-1} (inversion.cpp:93-102)
 * ride in the factorisation's graph, step i right after column i of L is in
 * place; otherwise the two passes run one after the other.  Results are
 * bit-identical either way; hk_timings()[1] / [2] = the LDLT proper and what
 * was left of L^{-1} after it. */
int hk_ldlt_invert(hk_ctx* ctx, int m);
int hk_get_Linv(hk_ctx* ctx, uint32_t* limbs, int32_t* exps, int32_t* signs);

/* k x k leading block of H^{-1} = sum_l Linv(l,j) Linv(l,c) / D_l, k <= m.
 * Replaces assemble_truncated_inverse (inversion.hpp:60) but keeps the block
 * in MP (no binary64 cast, inversion.cpp:258).  hk_get_block: k*k row-major. */
int hk_assemble_block(hk_ctx* ctx, int k);
int hk_get_block(hk_ctx* ctx, uint32_t* limbs, int32_t* exps, int32_t* signs);

/* s smallest eigenvalues of H from the last block: lambda_i = 1/mu_{k+1-i}
 * and trunc_err_i vs the (k-1) block.  Replaces smallest_eigs_of_H
 * (jacobi.hpp:29-30; jacobi.cpp:74-103).  Host cyclic Jacobi in binary128;
 * lambda = lambda_hi + lambda_lo (double-double, ~32 digits). */
int hk_smallest_eigs(hk_ctx* ctx, int s, double* lambda_hi, double* lambda_lo, double* trunc_err);

/* Host-only eigensolves (no context, no device):
 * hk_jacobi_eigenvalues — jacobi_eigenvalues(m, k, {tol_factor, max_sweeps})
 *   (jacobi.hpp:16-17): ascending eigenvalues of a symmetric k x k binary64
 *   block, cyclic Jacobi carried in binary128.  HK_ERR_RUNTIME on no convergence.
 * hk_block_eigenvalues — smallest_eigs_of_H (jacobi.hpp:29-30) on a k x k MP
 *   block given as host SoA (e.g. from hk_get_block): as hk_smallest_eigs. */
int hk_jacobi_eigenvalues(const double* m, int k, double tol_factor, int max_sweeps, double* out);
int hk_block_eigenvalues(int k, int limbs, const uint32_t* limbs_in, const int32_t* exps, const int32_t* signs, int s,
                         double* lambda_hi, double* lambda_lo, double* trunc_err);

/* Whole path, host buffers in, lambdas out: upload -> LDLT -> L^{-1} -> block
 * -> eigen.  Replaces hankel::compute (pipeline.hpp:50; pipeline.cpp:26-72)
 * with k clamped to n (pipeline.cpp:36) and s = min(3, k) (pipeline.cpp:64). */
int hk_compute(hk_ctx* ctx, int n, const uint32_t* limbs, const int32_t* exps, const int32_t* signs, int k,
               double* lambda_hi, double* lambda_lo, double* trunc_err, int* s_out);

/* The same path with the moments generated on the device (hk_generate_moments):
 * the inputs are the scalars of ComputeOptions (pipeline.hpp:13-26) only. */
int hk_compute_generated(hk_ctx* ctx, unsigned beta_num, unsigned beta_den, int n, int k, double* lambda_hi,
                         double* lambda_lo, double* trunc_err, int* s_out, int* moments_exact);

/* Stage times of the last calls, RunRecord taxonomy (pipeline.hpp:38-45), in
 * seconds: [0] wall (hk_compute), [1] ldlt, [2] invL, [3] invH, [4] eigen,
 * [5] h2d (or the on-device moment generation), [6] d2h.  Device stages are CUDA-event times on the ctx stream. */
int hk_timings(const hk_ctx* ctx, double* out7);

/* Kernel launches issued by the last hk_ldlt / invert / assemble calls. */
long long hk_launch_count(const hk_ctx* ctx);

/* Elementwise batch arithmetic on host SoA arrays (parity tests of the MP
 * kernels).  op = HK_OP_*.  a, b, c are `count`-long arrays (b, c unused as the
 * op requires; pass NULL). */
int hk_mp_batch(hk_ctx* ctx, int op, long long count, const uint32_t* a_l, const int32_t* a_e, const int32_t* a_s,
                const uint32_t* b_l, const int32_t* b_e, const int32_t* b_s, const uint32_t* c_l,
                const int32_t* c_e, const int32_t* c_s, uint32_t* o_l, int32_t* o_e, int32_t* o_s);

/* The context's CUDA stream (cudaStream_t as void*), so a caller can order
 * its own events / work with the path's kernels. */
void* hk_stream(const hk_ctx* ctx);

/* Measurement hook (no reference counterpart): run the LDLT once more,
 * eagerly on one stream, with CUDA events around every launch.  ms7 receives
 * the summed kernel milliseconds of [0] trailing update (the hot stage,
 * ldlt.cpp:122-129), [1] reciprocal, [2] B column, [3] L store, [4] the whole
 * eager LDLT, and on the tensor-core path the split of [0] into [5] limb
 * products (A preformat + k_tc_bulk) and [6] certified rounding (+ fix-ups);
 * *n_trailing the number of trailing steps. */
int hk_profile_ldlt(hk_ctx* ctx, double* ms7, long long* n_trailing);

/* Measurement hook: with hk_set_kernel_timing(ctx, 1) the captured LDLT graph
 * carries event-record nodes around every step's bulk kernels, and
 * hk_kernel_times returns, for the last hk_ldlt: out6[0] summed milliseconds of
 * the limb-product kernels (tensor-core A preformat + products, or the IMAD
 * trailing kernel), [1] of the certified rounding + fix-up pass, [2] the number
 * of timed steps; for a sharded context (always recorded) [3] summed ms of the
 * pivot-column broadcasts including the wait for their root — the reference's
 * WorkerTimings::comm_s (ldlt.cpp:214-263, 341) — and [4] their count; [5] the
 * LDLT's own time (ms). */
int hk_set_kernel_timing(hk_ctx* ctx, int on);

/* Test hook: how many items of the fused tensor-core rounding (csrc/tc_fused.cuh)
 * failed its final normalisation check since the context was created.  The
 * exponent prediction is certified, so this must stay 0; tests assert it. */
int hk_fused_violations(hk_ctx* ctx, long long* out);
/* Measurement hook: items the certified roundings (tensor-core paths) left to
 * the exact redo kernel since the context was created. */
int hk_fix_count(hk_ctx* ctx, long long* out);
int hk_kernel_times(hk_ctx* ctx, double* out6);
/* ... and per timed step s < cap: out[2s] product ms, out[2s+1] rounding + fix-up ms; *count steps. */
int hk_kernel_step_times(hk_ctx* ctx, double* out, int cap, int* count);

/* Measured integer-MAC peak of the device: 32x32->64-bit limb MACs per second
 * of the IMAD.WIDE carry chain the MP kernels use (register-only microkernel
 * over all SMs).  The roofline denominator for the IMAD path. */
int hk_peak_imad(int device, double* limb_macs_per_s);

/* Measured int8 tensor-core peak: u8 x u8 MACs per second of back-to-back
 * tcgen05.mma.kind::i8 (M=128, N=256, K=32, the product kernel's shape) on
 * every SM.  The roofline denominator for the tensor-core path (one limb-MAC
 * = 16 u8 MACs). */
int hk_peak_i8mma(int device, double* u8_macs_per_s);

/* ---- multi-GPU (one process per GPU) --------------------------
 * decompose_parallel's worker split (ldlt.hpp:97-99; W threads + slot channel,
 * ldlt.cpp:137-395) becomes `world` GPUs: rank r owns the columns
 * assign_columns(n, world) gives it, the pivot column is ncclBroadcast from its
 * owner every step, and after the factorisation the columns are gathered to
 * rank 0, which runs L^{-1} / block / eigen.  Results are bit-identical for any
 * world size.  hk_nccl_unique_id on rank 0, shared by the caller (e.g. over
 * torch.distributed), then hk_create_sharded on every rank (collective).
 * With nccl_id128 == NULL all `world` ranks are emulated inside this one
 * context on one device (broadcast = device-to-device copy): the sharded
 * kernels and maps, testable on a single GPU; rank must then be 0.
 * hk_compute returns rank 0's status and lambdas on every rank (one small
 * broadcast), so the callers' precision-search loops agree across ranks.
 * On a sharded context hk_invert_L_partial and hk_assemble_block are
 * collective too (every rank calls them): rows are owned in 128-row blocks
 * (block b on rank b % world), column i of L and row i of L^{-1} are broadcast
 * at step i (inversion.cpp:106-230, the per-row publish), and the block's
 * terms are reduced per rank up to 128-row subtrees of the fixed pairwise tree
 * that rank 0 finishes — results bit-identical to one GPU; rank 0 holds
 * L^{-1} and the block (hk_get_Linv / hk_get_block). */
int hk_nccl_unique_id(void* out128);
int hk_create_sharded(int device, int limbs, int rank, int world, const void* nccl_id128, hk_ctx** out);
int hk_world(const hk_ctx* ctx, int* rank, int* world);

/* A caller's column -> rank map for the sharded LDLT of order n (any map with
 * owners in [0, world); ColumnAssignment of decompose_parallel, ldlt.hpp:13-21,
 * 97-99 — the reference accepts any assignment, ldlt.cpp:355-395).  Without it
 * the context uses assign_columns(n, world).  Results do not depend on it. */
int hk_set_owner_map(hk_ctx* ctx, int n, const int32_t* owner);

/* Balanced round-robin (boustrophedon) ownership map, assign_columns
 * (ldlt.cpp:22-35): owner[c] for c < n. */
int hk_assign_columns(int n, int workers, int32_t* owner);

#ifdef __cplusplus
}
#endif

#endif /* HANKEL_B200_H */
