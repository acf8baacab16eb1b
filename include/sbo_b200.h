/*
 * sbo_b200.h — C ABI of the B200-native SBO iteration (arXiv 1412.4944).
 *
 * The library (paper_1412_4944_b200/libsbo_b200.so) exports the device
 * operations one Single-Block-Orthogonal dictionary-learning iteration is made
 * of.  Every entry point takes plain DEVICE pointers, sizes and a cudaStream_t
 * passed as void*; all work is stream-ordered and asynchronous.  No torch
 * types cross this boundary.  Each function names the reference function it
 * replaces (paths relative to /root/reference/pkg/src/orthodict/).
 *
 * Layouts (device):
 *   signals  y      : float32 or float64 (dtype), m rows of p  (signal j = y[j*p .. j*p+p-1]; this is the
 *                     reference's column-major p x m matrix, one contiguous column per signal)
 *   blocks   Q      : float64, K row-major p x p matrices (Q_b[k][i] = blocks[b*p*p + k*p + i];
 *                     atom i of block b is column i, exactly numpy's C-order block)
 *   codes  idx/val  : int16 / float64, k = min(s0, p) rows of a row stride `ld`
 *                     (row r, column j at r*ld + j; indices ascending down a column)
 *
 * Return value: SBO_OK or an error code; sbo_last_error() gives the message.
 * Numerical failures detected on the device (orthonormality defect > 1e-8,
 * Jacobi non-convergence) are reported through the int32 `status` arrays the
 * caller owns, so that a whole iteration can be enqueued without host syncs.
 */
#ifndef SBO_B200_H
#define SBO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SBO_OK = 0,
  SBO_EINVAL = 1,       /* bad argument              -> ValueError          */
  SBO_ENUMERICAL = 2,   /* defect > 1e-8             -> NumericalError      */
  SBO_EDECOMP = 3,      /* SVD/eig did not converge  -> DecompositionError  */
  SBO_ECUDA = 4         /* CUDA launch/runtime error -> RuntimeError        */
};

enum { SBO_KIND_SQUARED_SUM = 0, SBO_KIND_ABS_SUM = 1 }; /* sbo.py:31 */

/* element type of the signal matrix: float32 (the fast path; exact whenever the
 * caller's float64 signals are float32-representable) or float64 (bit-faithful
 * to arbitrary float64 inputs). */
enum { SBO_F32 = 0, SBO_F64 = 1 };

/* per-block device status words written by sbo_polar / sbo_init_block */
enum { SBO_ST_OK = 0, SBO_ST_SKIPPED = 1, SBO_ST_DEFECT = 2, SBO_ST_NOCONV = 3 };

int sbo_abi_version(void);
const char* sbo_last_error(void);
/* 1 when the calling process has a usable sm_100 device */
int sbo_device_ok(int device);

/* ---------------------------------------------------------------------------
 * Representation, energy pass — replaces sbo.py:177-194 (represent, pass 1) and
 * the per-block scoring of sbo.py:126-135 (block_energy).
 * For every signal j < m and block b in [b0, b1): c = Q_b^T y_j, score =
 * sum of the k largest c^2 (kind 0) or |c| (kind 1); the winner is the first
 * maximum.  accumulate = 0: fresh pass (b0 must be 0).  accumulate = 1: the
 * incoming (best, score, residual_sq) describe blocks [0, b0) and a block in
 * [b0, b1) replaces the winner only with a strictly larger score — the
 * incremental pass after a block is appended (sbo.py:357-363).
 * Outputs per signal: best block, its score, the winner's squared residual
 * ||y - Q_b x||^2 (the energy of the discarded coefficients; = ||y||^2 - kept by
 * Parseval, sbo.py:218, without the cancellation) and, optionally, ||y||^2.
 */
int sbo_energy_pass(const void* y, int dtype, int64_t m, int p, const double* blocks, int b0,
                    int b1, int s0, int kind, int accumulate, int32_t* best, double* score,
                    double* residual_sq, double* norm_sq, void* stream);

/* Exact float64 re-decision of the signals list[0 .. *nlist) over blocks [b0, K):
 * rewrites their best / score / residual_sq (the certification step after the
 * tensor-core energy pass flags near-ties).  b0 > 0 is the incremental form
 * (represent after a block was appended, sbo.py:361): the incoming best / score /
 * residual_sq stand for blocks < b0 and must be exact (sbo_residual_segments
 * writes exact scores); ties keep the lower block.  max_list bounds *nlist. */
int sbo_energy_recheck(const void* y, int dtype, int64_t m, int p, const double* blocks, int b0,
                       int K, int s0, int kind, const int32_t* list, const int32_t* nlist,
                       int64_t max_list, int32_t* best, double* score, double* residual_sq,
                       void* stream);

/* ---------------------------------------------------------------------------
 * Tensor-core energy pass, p = 64 (tc_energy.cu) — the same contract as
 * sbo_energy_pass on split-fp16 operands with fp32 accumulation in TMEM:
 *   sbo_tc_split_signals: y -> yh, yl (fp16 hi/lo, 128-B rows pre-swizzled) and a
 *     per-signal power-of-two scale; arrays sized sbo_tc_padded_rows(m) rows.
 *   sbo_tc_split_blocks:  K blocks -> qh, ql (atom rows, pre-swizzled) + scales.
 *   sbo_tc_energy: best block per signal with an error-bounded certificate;
 *     signals whose decision is within the bound are appended to flags
 *     (count in *nflag, which the caller zeroes) for sbo_energy_recheck.
 *     score / residual_sq of unflagged signals are float32-accurate.
 */
int64_t sbo_tc_padded_rows(int64_t m);
int sbo_tc_split_signals(const void* y, int dtype, int64_t m, int p, void* yh, void* yl,
                         int16_t* escale, void* stream);
int sbo_tc_split_blocks(const double* Q, int K, int p, void* qh, void* ql, int16_t* fscale,
                        void* stream);
int sbo_tc_energy(const void* yh, const void* yl, const int16_t* escale, int64_t m,
                  const void* qh, const void* ql, const int16_t* fscale, int b0, int b1, int s0,
                  int kind, int accumulate, int32_t* best, double* score, double* residual_sq,
                  int32_t* flags, int32_t* nflag, uint64_t* cand, void* stream);
/* p = 256 (config D), s0 <= 32: the same contract as sbo_tc_energy on operands
 * from sbo_tc_split_signals / sbo_tc_split_blocks with p = 256 (tc_energy256.cu). */
int sbo_tc_energy256(const void* yh, const void* yl, const int16_t* escale, int64_t m,
                     const void* qh, const void* ql, const int16_t* fscale, int b0, int b1,
                     int s0, int kind, int accumulate, int32_t* best, double* score,
                     double* residual, int32_t* flags, int32_t* nflag, uint64_t* cand,
                     void* stream);

/* Candidate blocks of the flagged signals (cand, optional, parallel to flags):
 * bit b - b0 set for every block whose approximate decision value was within
 * the certificate's tolerance of the best (b1 - b0 <= 64; the p = 256 pass sets
 * every bit above 32 blocks) — a
 * superset of the blocks that can win in float64.  sbo_cand_sort orders the
 * flag list by its two lowest candidate blocks, so that tiles of the float64
 * re-decision share few blocks (order within a group is arbitrary: each
 * signal's decision is independent of it).  Workspace: sbo_cand_workspace_bytes. */
size_t sbo_cand_workspace_bytes(void);
int sbo_cand_sort(const int32_t* flags, const uint64_t* cand, const int32_t* nflag,
                  int64_t max_list, int32_t* flags_out, uint64_t* cand_out, void* ws,
                  size_t ws_bytes, void* stream);

/* sbo_energy_recheck restricted per tile to the union of the listed signals'
 * candidate blocks (cand parallel to list; blocks b0 + bit), b1 - b0 <= 64. */
int sbo_energy_recheck_cand(const void* y, int dtype, int64_t m, int p, const double* blocks,
                            int K, int s0, int kind, const int32_t* list, const uint64_t* cand,
                            const int32_t* nlist, int64_t max_list, int32_t* best, double* score,
                            double* residual_sq, void* stream);

/* ---------------------------------------------------------------------------
 * Stable grouping by block — replaces sbo.py:231-249 (group_by_block) and the
 * argsort/searchsorted of sbo.py:200-201.  perm lists signals block by block,
 * original order inside a block; bounds[b] .. bounds[b+1] is block b's range.
 * Also emits the segment table used by the per-block kernels: every block's
 * range split into chunks of at most `seg_len` signals (seg_len multiple of 64).
 * Workspace: sbo_group_workspace_bytes(m, K).
 */
size_t sbo_group_workspace_bytes(int64_t m, int K);
int64_t sbo_max_segments(int64_t m, int K, int seg_len);
int sbo_group(const int32_t* best, int64_t m, int K, int seg_len, int32_t* perm,
              int64_t* bounds, int32_t* seg_block, int64_t* seg_lo, int64_t* seg_hi,
              int32_t* nseg, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Own-block coding — replaces onb.py:58-76 (select_top) applied to Q_b^T y as in
 * sbo.py:203-209 (represent pass 2) and onb.py:170 (train_onb coding step).
 * Segments from sbo_group (or a single segment over a member list).  For the
 * signal at order[t] (t in a segment of block b): its k kept indices (ascending)
 * and values are written at column `t` (out_by_signal = 0) or at column
 * order[t] (out_by_signal = 1) of idx/val (row stride ld).  energy/residual_sq
 * (optional, indexed like the codes) receive the score of the kept values and
 * the squared residual (sbo.py:213-218).  block_override >= 0 codes every segment
 * against that block instead of seg_block.
 */
int sbo_code_segments(const void* y, int dtype, int p, const int32_t* order, const int32_t* seg_block,
                      const int64_t* seg_lo, const int64_t* seg_hi, const int32_t* nseg,
                      int64_t max_seg, const double* blocks, int block_override, int s0,
                      int kind, int out_by_signal, int64_t ld, int16_t* idx, double* val,
                      double* energy, double* residual_sq, void* stream);

/* ---------------------------------------------------------------------------
 * Sparse outer product P = Y X^T per segment — replaces onb.py:127-134
 * (sparse_outer).  Codes are read at column t of the segment order (the layout
 * sbo_code_segments writes with out_by_signal = 0).  partial receives one
 * float64 p x p matrix per segment (row-major, P[k][i] = sum y[k] x[i]);
 * sbo_reduce_segments sums the partials of each block in segment order
 * (deterministic) into P (K x p x p).  counts (optional, K int64) receives
 * bounds-derived signal counts per block.
 */
int sbo_outer_segments(const void* y, int dtype, int p, const int32_t* order, const int64_t* seg_lo,
                       const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg, int s0,
                       int64_t ld, const int16_t* idx, const double* val, double* partial,
                       void* stream);
int sbo_reduce_segments(const double* partial, const int32_t* seg_block, const int32_t* nseg,
                        int64_t max_seg, int K, int p, double* P, void* stream);

/* Fused 1ONB round for p <= 64, any s0 — onb.py:170-171 (coding of
 * every signal in its own block, then P = Y X^T) in one pass per segment: the
 * same partials as sbo_code_segments + sbo_outer_segments, codes not stored. */
int sbo_round_segments(const void* y, int dtype, int p, const int32_t* order,
                       const int32_t* seg_block, const int64_t* seg_lo, const int64_t* seg_hi,
                       const int32_t* nseg, int64_t max_seg, const double* blocks,
                       int block_override, int s0, double* partial, void* stream);

/* Coding half of a 1ONB round for p <= 64 (onb.py:170 select_top(Q^T Y)): the
 * fused round's float64 projection and exact selection, writing the kept pairs
 * of every signal at column t of the segment order (idx/val rows of stride ld,
 * the layout of sbo_code_segments with out_by_signal = 0) for
 * sbo_outer_i8_segments. */
int sbo_round_code_segments(const void* y, int dtype, int p, const int32_t* order,
                            const int32_t* seg_block, const int64_t* seg_lo,
                            const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                            const double* blocks, int block_override, int s0, int64_t ld,
                            int16_t* idx, double* val, void* stream);

/* The 1ONB round's coding (onb.py:170-171: select_top(Q^T Y)) and represent's
 * residual pass (sbo.py:207-218) for p = 64, 1 <= s0 <= 32, on the tcgen05
 * tensor cores: the projection is computed exactly from integer digits
 * (tcgen05.mma kind::i8; y as the sbo_y_digits rows, y = Y_int 2^-sy; each
 * block entry rounded to 2^-54 in 8 digits; digit levels of weight >= 2^-49
 * relative kept), then the exact top-s0 selection (ties -> lower atom).
 * Replaces the DMMA projection of sbo_round_code_segments /
 * sbo_residual_segments.  Segments as sbo_round_code_segments; blocks holds
 * nblocks blocks (block_override >= 0: every segment uses that block).
 * mode 0 (code): the kept pairs of position t at column t of idx/val (stride ld);
 * mode 1 (resid): rest_sq[order[t]] = energy of the discarded coefficients,
 * score[order[t]] (optional) = the kept score of `kind`.
 * Workspace: sbo_round_i8_workspace_bytes(nblocks). */
size_t sbo_round_i8_workspace_bytes(int nblocks);
int sbo_round_i8_segments(const void* ydig, int sy, const int32_t* order,
                          const int32_t* seg_block, const int64_t* seg_lo,
                          const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                          const double* blocks, int nblocks, int block_override, int s0,
                          int mode, int kind, int64_t ld, int16_t* idx, double* val,
                          double* rest_sq, double* score, void* workspace, size_t ws_bytes,
                          void* stream);

/* Sparse outer products P = Y X^T per block on the tcgen05 tensor cores
 * (onb.py:127-134; north_star "grouped GEMM Y_j X_j^T"), p = 64 or 256, float32
 * signals: y (as the transposed digit tiles of sbo_y_tiles, built once per
 * grouping) and the code values cut into
 * 7-bit integer digits (y = Y_int 2^-sy exactly, 5 digits; x rounded to the
 * 2^-sx grid, 8 digits), digit products accumulated exactly in int32 TMEM and
 * int64 global accumulators (levels of weight >= 2^-49 relative kept), so P
 * is independent of the signal order and the segmentation.  P receives
 * nblocks x p x p float64 (P[b][k][i] = sum y[k] x[i] over the signals of the
 * segments with seg_block = b; seg_block NULL = every segment in block 0) —
 * the result sbo_reduce_segments would give.  Codes are read at column t of
 * the segment order (sbo_round_code_segments).  sy / sx come from sbo_i8_scan:
 * every |y| < 2^(35 - sy) on the 2^-sy grid, every |x| < 2^(54 - sx).
 * p = 256 runs the p = 64 product on each of the 16 (64-dim, 64-atom) slices.
 * Workspace: sbo_outer_i8_workspace_bytes(nblocks, p). */
size_t sbo_outer_i8_workspace_bytes(int nblocks, int p);
int sbo_outer_i8_segments(const void* ytiles, int p, const int32_t* seg_block,
                          const int64_t* seg_lo,
                          const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                          int nblocks, int s0, int64_t ld, const int16_t* idx,
                          const double* val, int sy, int sx, double* P, void* workspace,
                          size_t ws_bytes, void* stream);

/* Transposed digit tiles of a segment table for sbo_outer_i8_segments: per
 * (segment, 128-position chunk) in segment order, the 5 digit planes of the
 * signals order[t] as [64 dims][128 signals] int8 (40 KB, the kernel's shared
 * memory image; p = 256: four such images per chunk, one per 64-dim group).
 * tiles: sbo_y_tiles_bytes(n, max_seg, p) bytes (n = positions). */
size_t sbo_y_tiles_bytes(int64_t n, int64_t max_seg, int p);
int sbo_y_tiles(const void* ydig, int p, const int32_t* order, const int64_t* seg_lo,
                const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg, void* tiles,
                void* stream);

/* Signal-major digit rows of float32 signals (p = 64 or 256) for
 * sbo_outer_i8_segments / sbo_round_i8_segments / sbo_coef_i8_segments: row s
 * (5 p bytes) = the 5 digit planes Y_a (p dims each) of y_s = Y_int 2^-sy. */
int sbo_y_digits(const void* y, int dtype, int64_t m, int p, int sy, void* ydig, void* stream);

/* Digit-format scan of float32 signals (m rows of p): out[0] = smallest E with
 * every |y| < 2^E, out[1] = smallest exponent of a set mantissa bit among the
 * nonzero values, out[2..3] = largest ||y||^2 as float64 bits. */
int sbo_i8_scan(const void* y, int dtype, int64_t m, int p, int32_t* out, void* stream);

/* Squared residuals of represent (sbo.py:213-218) for p <= 64, any s0:
 * every signal of a segment is coded in its segment's block in float64 (exact
 * selection, as sbo_code_segments) and rest_sq[order[t]] receives the energy of
 * its discarded coefficients; score (optional) the exact energy of the kind
 * (block_energy, sbo.py:126-135).  Replaces sbo_code_segments(idx = val = NULL). */
int sbo_residual_segments(const void* y, int dtype, int p, const int32_t* order,
                          const int32_t* seg_block, const int64_t* seg_lo, const int64_t* seg_hi,
                          const int32_t* nseg, int64_t max_seg, const double* blocks, int s0,
                          int kind, double* rest_sq, double* score, void* stream);

/* ---------------------------------------------------------------------------
 * Gram matrix G = Y_W Y_W^T of a member list (float64) — the data term of the
 * new block's initialisation (onb.py:79-95 via thin_svd(ysub), linalg.py:52).
 * Partials: one p x p matrix per chunk of `chunk` members, reduced in order.
 * Workspace: sbo_gram_workspace_bytes(w, chunk, p).
 */
size_t sbo_gram_workspace_bytes(int64_t w, int chunk, int p);
int sbo_gram(const void* y, int dtype, int p, const int32_t* members, int64_t w, int chunk,
             double* G, void* ws, size_t ws_bytes, void* stream);
/* sbo_gram over the first min(w, *count) members, count read on the device (a
 * sharded worst set's local member count stays in device memory; w sizes the
 * workspace and launches). */
int sbo_gram_counted(const void* y, int dtype, int p, const int32_t* members, int64_t w,
                     const int64_t* count, int chunk, double* G, void* ws, size_t ws_bytes,
                     void* stream);
/* Segment table of a list of min(w, *count) entries (count NULL: w) in chunks
 * of `chunk`: seg_lo/seg_hi (ceil(w / chunk) entries), *nseg = the used count. */
int sbo_chunk_segments(int64_t w, const int64_t* count, int chunk, int64_t* seg_lo,
                       int64_t* seg_hi, int32_t* nseg, void* stream);

/* select_top on explicit float64 coefficient vectors (onb.py:58-76): vector j
 * is row j of coeffs (t x p); codes written at column j (row stride ld). */
int sbo_select_top(const double* coeffs, int64_t t, int p, int s0, int64_t ld, int16_t* idx,
                   double* val, void* stream);

/* The coding step of sbo_code_segments (sbo.py:196-211, onb.py:170) on
 * coefficient rows computed by sbo_coef_i8_segments: row j (p doubles) is
 * position j < min(t, *n) (n NULL: t) of a segment table; its outputs go to
 * column order[j] (order NULL: j) — the kept pairs (idx/val, stride ld; both
 * NULL to skip), energy[col] = the kept score of `kind`, rest_sq[col] = the
 * energy of the discarded coefficients (each optional).  Exact selection,
 * ties -> lower atom. */
int sbo_select_coded(const double* coeffs, const int64_t* n, int64_t t, int p, int s0, int kind,
                     const int32_t* order, int64_t ld, int16_t* idx, double* val,
                     double* energy, double* rest_sq, void* stream);

/* Coefficients C = Q^T y for p = 256 (the projection of sbo_code_segments,
 * onb.py:170) on the tcgen05 tensor cores from integer digits (tcgen05.mma
 * kind::i8): y as the sbo_y_digits rows (p = 256, y = Y_int 2^-sy), each block
 * entry rounded to 2^-54 in 8 digits, digit levels of weight >= 2^-49 relative
 * kept, exact int32 sums in TMEM.  coef row t (256 float64) = the coefficients
 * of signal order[t] (order NULL: t) in its segment's block (block_override >=
 * 0: that block) for every position t a segment covers.  Segments as
 * sbo_code_segments; blocks holds nblocks blocks.
 * Workspace: sbo_coef_i8_workspace_bytes(nblocks). */
size_t sbo_coef_i8_workspace_bytes(int nblocks);
int sbo_coef_i8_segments(const void* ydig, int sy, const int32_t* order,
                         const int32_t* seg_block, const int64_t* seg_lo, const int64_t* seg_hi,
                         const int32_t* nseg, int64_t max_seg, const double* blocks, int nblocks,
                         int block_override, double* coef, void* workspace, size_t ws_bytes,
                         void* stream);

/* The float64 re-decision of flagged signals (the role of
 * sbo_energy_recheck_cand, same arguments and outputs) for p = 256 with the
 * projection of sbo_coef_i8_segments: list[0 .. *nlist) sorted by candidate
 * mask (sbo_cand_sort), cand[i] = the candidate blocks of list[i] (K <= 64);
 * each signal's energy (sbo.py:126-135, exact selection) in each of its
 * candidate blocks, the first maximum wins (ties -> lower block, sbo.py:191);
 * best / score / residual of list[i] are overwritten.  ydig / sy as
 * sbo_coef_i8_segments.  Workspace: sbo_recheck_i8_workspace_bytes(K) (for the
 * current device). */
size_t sbo_recheck_i8_workspace_bytes(int K);
int sbo_energy_recheck_i8(const void* ydig, int sy, const double* blocks, int K, int s0, int kind,
                          const int32_t* list, const uint64_t* cand, const int32_t* nlist,
                          int64_t max_list, int32_t* best, double* score, double* residual,
                          void* workspace, size_t ws_bytes, void* stream);

/* sbo_energy_recheck_i8 (same arguments and outputs) over (signal, candidate
 * block) pairs: the flagged signals are bucketed per candidate block and each
 * block's list is projected (sbo_coef_i8_segments) and ranked
 * (sbo_select_coded) alone, so only the pairs the masks name are computed; the
 * first maximum over each signal's candidates in ascending block order wins.
 * list need not be sorted.  Workspace: sbo_recheck_pairs_workspace_bytes(K,
 * max_list). */
size_t sbo_recheck_pairs_workspace_bytes(int K, int64_t max_list);
int sbo_energy_recheck_pairs(const void* ydig, int sy, const double* blocks, int K, int s0,
                             int kind, const int32_t* list, const uint64_t* cand,
                             const int32_t* nlist, int64_t max_list, int32_t* best,
                             double* score, double* residual, void* workspace, size_t ws_bytes,
                             void* stream);

/* ---------------------------------------------------------------------------
 * Polar update Q_b = U V^T of P_b for the blocks whose count > 0 — replaces
 * linalg.py:68-78 (procrustes_polar via thin_svd/gesdd) and the guard of
 * onb.py:119-124.  One-sided Jacobi (Hestenes) in float64.  Q (K x p x p) is
 * updated in place; blocks with counts[b] == 0 (counts may be NULL) are left
 * unchanged and flagged SBO_ST_SKIPPED (sbo.py:379-383).  V (optional, K x p x p
 * column-major, in/out) warm-starts the rotation from the previous round's
 * right singular vectors and receives the new ones (the identity is a valid
 * first guess).  sigma (optional, K x p) receives the singular values in
 * descending order.  status[b]: low byte SBO_ST_*, bits 8..15 sweeps used.
 * Workspace: sbo_polar_workspace_bytes(K, p).
 */
size_t sbo_polar_workspace_bytes(int K, int p);
int sbo_polar(const double* P, int K, int p, const int64_t* counts, double* Q, double* V,
              double* sigma, int32_t* status, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * New block initialisation from a Gram matrix — replaces onb.py:79-116
 * (init_onb + _complete_columns) with thin_svd's canonical signs
 * (linalg.py:32-37).  Eigenvectors of G in descending eigenvalue order, each
 * column's largest-|entry| made nonnegative; directions with
 * sqrt(lambda_i) <= 1e-12 sqrt(lambda_0) — or below the float64 resolution of
 * the Gram route, lambda_i <= 64 eps lambda_0 — are replaced by the twice-
 * projected Gram–Schmidt completion against the host-drawn normals `draws`
 * (ndraws x p, the block stream's standard_normal draws in order).
 * ncols < p (fewer members than dimensions) keeps at most ncols directions.
 * rank (optional, 2 x int32) receives the number of kept directions and the
 * number of completion draws consumed.
 */
size_t sbo_init_workspace_bytes(int p);
int sbo_init_block(const double* G, int p, int64_t ncols, const double* draws, int ndraws,
                   double* Q, int32_t* rank, int32_t* status, void* ws, size_t ws_bytes,
                   void* stream);

/* ---------------------------------------------------------------------------
 * Thin SVD of a rows x cols float64 matrix with rows >= cols (callers transpose
 * wide inputs) — replaces linalg.py:40-65 (thin_svd: gesdd/gesvd + canonical
 * signs).  Outputs row-major U (rows x cols), S (cols, descending) and
 * V (cols x cols) with A = U diag(S) V^T.  status: SBO_ST_OK / SBO_ST_NOCONV.
 */
size_t sbo_svd_workspace_bytes(int rows, int cols);
int sbo_svd(const double* A, int rows, int cols, double* U, double* S, double* V,
            int32_t* status, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Worst-represented set — replaces sbo.py:223-228 (worst_set).  The members of
 * the w largest residual_sq (ties toward low signal index), written in
 * ascending signal order to members[0 .. min(w, m)).  Radix select on the
 * float64 keys.  Workspace: sbo_worst_workspace_bytes(m).
 * The split form exposes the radix passes for a multi-GPU select: a histogram
 * of the 256 digit values at `shift` among keys whose bits above shift+8 equal
 * `prefix` (key_hist), and the final member compaction given the threshold key
 * and the number of threshold-equal members to keep (worst_collect).
 */
size_t sbo_worst_workspace_bytes(int64_t m);
int sbo_worst_set(const double* residual_sq, int64_t m, int64_t w, int32_t* members,
                  void* ws, size_t ws_bytes, void* stream);
int sbo_key_histogram(const double* residual_sq, int64_t m, uint64_t prefix, int shift,
                      int64_t* hist256, void* stream);
int sbo_worst_collect(const double* residual_sq, int64_t m, uint64_t threshold_key,
                      int64_t take_equal, int32_t* members, int64_t* count, void* ws,
                      size_t ws_bytes, void* stream);
/* Device-resident form of the sharded select (no host round trip): begin sets
 * the state in ws (need = global worst-set size); per shift 56, 48, .., 0 the
 * caller runs select_hist, allreduces hist256 across ranks (device memory,
 * NCCL) and runs select_pick; select_counts writes this rank's (greater, equal)
 * counts against the threshold to gt_eq[2]; the caller allgathers gt_eq[1]
 * into eq_all[world]; select_write keeps the threshold ties of lower ranks
 * first (dist.equal_quota) and writes the members and their count[1]. */
int sbo_select_begin(void* ws, int64_t need, void* stream);
int sbo_select_hist(const double* residual_sq, int64_t m, void* ws, int shift, int64_t* hist256,
                    void* stream);
int sbo_select_pick(void* ws, int64_t* hist256, int shift, void* stream);
int sbo_select_counts(const double* residual_sq, int64_t m, void* ws, size_t ws_bytes,
                      int64_t* gt_eq, void* stream);
int sbo_select_write(const double* residual_sq, int64_t m, void* ws, size_t ws_bytes,
                     const int64_t* gt_eq, const int64_t* eq_all, int rank, int32_t* members,
                     int64_t* count, void* stream);

/* ---------------------------------------------------------------------------
 * Deterministic float64 sum (fixed tree) — sbo.py:295-296 (_rmse numerator).
 */
size_t sbo_sum_workspace_bytes(int64_t n);
int sbo_sum(const double* x, int64_t n, double* total, void* ws, size_t ws_bytes, void* stream);

/* ||Q_b^T Q_b - I||_F for K blocks (linalg.py:81-86). */
int sbo_defect(const double* Q, int K, int p, double* out, void* stream);

/* Exact reconstruction error sum_j ||y_j - Q_{b_j} x_j||^2 (linalg.py:148-162). */
int sbo_frobenius_sq(const void* y, int dtype, int64_t m, int p, const double* blocks,
                     const int32_t* block, int s0, int64_t ld, const int16_t* idx,
                     const double* val, double* total, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Signal ingestion — replaces data.py:182-208 (extract_patches) after its corner
 * draws (rows[j], cols[j]: numpy default_rng(seed).integers on the host).  Writes
 * count rows of edge^2 entries: entry c*edge + r of row j is
 * grid[(rows[j] + r) * ld + cols[j] + c] / 255 (float64), minus the patch mean
 * (numpy's pairwise float64 sum / edge^2) for normalization 1
 * ("unit-range-dc-removed").  grid_dtype: 0 uint8, 1 float64; out_dtype SBO_F32
 * (round-to-nearest of the float64 value) or SBO_F64.  edge <= 32.  A uint8 grid
 * is read in aligned 4-byte words: its allocation must be 4-byte aligned and
 * padded to a multiple of 4 bytes (cudaMalloc and the torch allocator are).
 */
int sbo_extract_patches(const void* grid, int grid_dtype, int64_t h, int64_t w, int64_t ld,
                        int edge, const int32_t* rows, const int32_t* cols, int64_t count,
                        int normalization, int out_dtype, void* out, void* stream);

/* ---------------------------------------------------------------------------
 * Codes persistence — the float64 payloads of store.py:99-115 (save_sbo_codes)
 * for signals [j0, j0 + n), written contiguously to out: record 0 = block as
 * float64 (n values), 1 = indices as float64 and 2 = values, each k per signal
 * (the column-major k x m payload of data.py:232-237).  indices / values are the
 * device code layout (k rows of stride ld).  Records 3 (energy) and 4
 * (residual_sq) are the device float64 arrays as they are.
 */
int sbo_codes_pack(int record, const int32_t* block, const int16_t* indices, const double* values,
                   int64_t ld, int k, int64_t j0, int64_t n, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SBO_B200_H */
