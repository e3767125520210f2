/*
 * libbamg_b200 -- C ABI of the B200-native LM linear-solve path of arXiv 2007.01941.
 *
 * The reference (`/root/reference/pkg/src/bamg`, Python + numpy/scipy) has no
 * native boundary of its own: every entry point below replaces a reference Python
 * function (cited file:line) whose arithmetic ran in numpy / scipy.sparse / LAPACK.
 * All pointers are DEVICE pointers unless named *_host; sizes are element counts;
 * `stream` is a cudaStream_t (NULL = legacy default stream). Buffers are owned by
 * the caller; the library allocates only stream-ordered scratch inside a call and
 * the small workspace in `bamg_ctx`.
 *
 * Return value: 0 = ok, >0 = domain error (see the BAMG_ERR_* codes; index
 * out-parameters carry details), <0 = CUDA / launch error. `bamg_last_error`
 * returns the thread-local message of the last failure.
 *
 * Layout: observations are stored point-major (sorted by (point, camera));
 * `cm_list` gives the point-major position of each observation in (camera, point)
 * order (the reference's W block order). Block matrices are BSR with int32
 * row pointers / column indices sorted per row and row-major fp64 blocks.
 */
#ifndef BAMG_B200_H
#define BAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BAMG_ABI_VERSION 1

#define BAMG_OK 0
#define BAMG_ERR_INDEFINITE 1   /* IndefiniteBlockError (blockmat.py:25-39) */
#define BAMG_ERR_BEHIND 2       /* BehindCameraError (problem.py:28-36) */
#define BAMG_ERR_NOT_PD 3       /* coarsest operator not PD (multigrid.py:434-440) */
#define BAMG_ERR_UNSUPPORTED 4  /* size outside the kernels' supported range */
#define BAMG_ERR_FORMAT 5       /* BalFormatError (balio.py:17-22): *err_line + message */
#define BAMG_ERR_CUDA (-1)

typedef struct bamg_ctx bamg_ctx;

int bamg_version(void);
bamg_ctx* bamg_ctx_create(void);
void bamg_ctx_destroy(bamg_ctx* ctx);
int bamg_last_error(char* buf, size_t n);

/* ---- primitives (replace numpy lexsort / cumsum / dot used across the path) ---- */
int bamg_scan_exclusive_i32(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int32_t* total,
                            void* stream);
int bamg_sort_pairs_u32(bamg_ctx* ctx, const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                        uint32_t* vout, int64_t n, int key_bits, void* stream);
int bamg_segment_ptr(bamg_ctx* ctx, const int32_t* sorted_ids, int64_t n, int32_t nseg, int32_t* ptr,
                     void* stream);
int bamg_gather_rows_f64(bamg_ctx* ctx, const double* src, const int32_t* idx, int64_t n, int32_t width,
                         double* dst, void* stream);
int bamg_scatter_rows_f64(bamg_ctx* ctx, const double* src, const int32_t* idx, int64_t n, int32_t width,
                          double* dst, void* stream);
int bamg_gather_i32(bamg_ctx* ctx, const int32_t* src, const int32_t* idx, int64_t n, int32_t* dst,
                    void* stream);
int bamg_dot(bamg_ctx* ctx, const double* x, const double* y, int64_t n, double* out_dev, void* stream);
int bamg_absmax(bamg_ctx* ctx, const double* x, int64_t n, double* out_dev, void* stream);
int bamg_axpby(bamg_ctx* ctx, double a, const double* x, double b, double* y, int64_t n, void* stream);
int bamg_negate(bamg_ctx* ctx, const double* a, double* b, int64_t n, void* stream);

/* ---- observation structure (problem.py:81-107 keeps input order; this is the
 *      device layout) and covisibility (schur.py:147-159, multigrid.py:52-80) ---- */
int bamg_obs_orders(bamg_ctx* ctx, const int32_t* cam_idx, const int32_t* pt_idx, int64_t k, int32_t nc,
                    int32_t npt, int32_t* pm_perm, int32_t* obs_cam_pm, int32_t* obs_pt_pm, int32_t* pt_ptr,
                    int32_t* cm_list, int32_t* cam_ptr, void* stream);
int bamg_covis_count(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* obs_pt_pm,
                     const int32_t* pt_ptr, const int32_t* obs_cam_pm, int32_t nc, int32_t* row_counts,
                     void* stream);
int bamg_covis_fill(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* obs_pt_pm,
                    const int32_t* pt_ptr, const int32_t* obs_cam_pm, int32_t nc, const int32_t* S_ptr,
                    int32_t* S_col, void* stream);
/* count pass that keeps each row's bitmap (nc x ceil(nc/32) words) for the fill */
int bamg_covis_count_keep(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* obs_pt_pm,
                          const int32_t* pt_ptr, const int32_t* obs_cam_pm, int32_t nc, int32_t* row_counts,
                          uint32_t* bitmaps, void* stream);
/* S columns from the kept bitmaps (replaces the fill pass's second sweep) */
int bamg_covis_compact(bamg_ctx* ctx, const uint32_t* bitmaps, int32_t nc, const int32_t* S_ptr, int32_t* S_col,
                       void* stream);
int bamg_shared_counts(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* obs_pt_pm,
                       const int32_t* pt_ptr, const int32_t* obs_cam_pm, int32_t nc, const int32_t* S_ptr,
                       const int32_t* S_col, int32_t max_row, int32_t* shared_cnt, void* stream);
/* multigrid.py:52-80 visibility_strength; flags_dev[0] = cameras with no points,
 * flags_dev[1] = int8-wrapped covisibility block count (schur.py:151-159). */
int bamg_visibility_strength(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* S_ptr, const int32_t* S_col,
                             const int32_t* shared_cnt, int32_t nc, int32_t* deg, int32_t* G_ptr, int32_t* G_col,
                             double* G_val, int32_t* flags_dev, void* stream);

/* ---- residuals / Jacobians: problem.py:202-219 (_project_arrays), 272-326 (evaluate) ---- */
/* J: (k, 32) observation records [F 2x9 | E 2x3 | H 2x3 | r 2] (H filled by build_system) */
int bamg_evaluate(bamg_ctx* ctx, const double* cams, int32_t nc, const double* pts, const int32_t* obs_cam,
                  const int32_t* obs_pt, const double* pixels, int64_t k, int32_t huber, int32_t with_jacobian,
                  double* J, double* w, uint8_t* behind, double* objective_dev, int32_t* n_behind_dev,
                  void* stream);

/* ---- normal blocks / damping / reduced system: problem.py:255-269, schur.py:38-47, 99-125 ---- */
int bamg_normal_blocks(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* pt_ptr,
                       const double* J, int32_t nc, int32_t npt, double* A_raw, double* g_cam, double* C_raw,
                       double* g_pt, void* stream);
int bamg_damping(bamg_ctx* ctx, const double* A_raw, const double* C_raw, int32_t nc, int32_t npt, double radius,
                 double* d_cam, double* d_pt, void* stream);
int bamg_build_system(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* pt_ptr,
                      double* J, int64_t k, const double* A_raw, const double* C_raw, const double* g_cam,
                      const double* g_pt, const double* d_cam, const double* d_pt, int32_t nc, int32_t npt,
                      double* A, double* C, double* Cinv, double* Cb, double* qo, double* rhs,
                      int32_t* bad_min_dev, void* stream);
/* A = A_raw + diag(d) (bs x bs blocks): the damped camera blocks, formed on demand */
int bamg_add_block_diag(bamg_ctx* ctx, const double* raw, const double* d, int32_t n, int32_t bs, double* out,
                        void* stream);
/* One camera-major pass over the records (schur.py:38-47, 99-125, 128-144): dA = diag(sum F^T F)
 * (dA_raw, optional), D = clip(dA, 1e-6, 1e32) / radius (d_cam, optional), and with S != NULL the
 * diagonal blocks S[dpos[i]] = sum F^T (I - H E^T) F + D and rhs = -sum F^T (r + q) (optional). */
int bamg_camera_pass(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J, const double* qo,
                     int32_t nc, double radius, const int32_t* dpos, double* S, double* rhs, double* d_cam,
                     double* dA_raw, void* stream);
/* rhs == NULL in bamg_build_system skips the right-hand side (formed later by
 * bamg_rhs_gather, or by bamg_schur_numeric's diagonal pass in the same sweep) */
int bamg_rhs_gather(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J, const double* qo,
                    const double* g_cam, int32_t nc, double* rhs, void* stream);
/* recompute the H slots of J (and q) from a system's C^-1 / C^-1 b */
int bamg_obs_H(bamg_ctx* ctx, const int32_t* obs_pt_pm, const double* Cinv, const double* Cb, int64_t k, double* J,
               double* qo, void* stream);
/* schur.py:84-86 implicit_matvec */
int bamg_implicit_matvec(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* pt_ptr,
                         const int32_t* obs_cam_pm, const double* J, const double* A, const double* Cinv,
                         const double* x, int32_t nc, int32_t npt, double* qo, double* y, void* stream);
/* schur.py:171-173 back_substitute */
int bamg_back_substitute(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm, const double* J,
                         const double* Cinv, const double* grad_pt, const double* dc, int32_t nc, int32_t npt,
                         double* dp, void* stream);
/* schur.py:114-116 W blocks in reference BSR order (API view) */
int bamg_materialize_W(bamg_ctx* ctx, const int32_t* cm_list, const double* J, int64_t k, double* W,
                       void* stream);

/* ---- explicit S: schur.py:128-144 (+ blockmat.py:308-353) ---- */
int bamg_schur_symbolic_sizes(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* S_ptr, const int32_t* S_col,
                              int32_t nc, int32_t npt, int32_t* pair_off, int32_t* dpos, int32_t* up_off,
                              int64_t* out_host, void* stream);
int bamg_schur_symbolic(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm, const int32_t* obs_pt_pm,
                        const int32_t* S_ptr,
                        const int32_t* S_col, int32_t nc, int32_t npt, int64_t nnz, const int32_t* pair_off,
                        int64_t n_pairs, const int32_t* dpos, const int32_t* up_off, int32_t* pair_a,
                        int32_t* pair_b, int32_t* blk_pair_ptr, int32_t* up_blk, int32_t* up_row,
                        int32_t* up_tpos, void* stream);
/* shared-point counts per S slot from the pair lists (list lengths, mirrored;
 * diagonal = camera degree): the strength pass without a sweep of the observations */
int bamg_shared_from_pairs(bamg_ctx* ctx, const int32_t* up_blk, const int32_t* up_tpos, int32_t n_up,
                           const int32_t* blk_pair_ptr, const int32_t* dpos, const int32_t* cam_ptr, int32_t nc,
                           int32_t* shared_cnt, void* stream);
/* reorder the upper-block work list by descending pair count (load balance) */
int bamg_schur_order_upper(bamg_ctx* ctx, int32_t* up_blk, int32_t* up_row, int32_t* up_tpos, int32_t n_up,
                           const int32_t* blk_pair_ptr, const int32_t* pair_a, void* stream);
/* row-owned variant: no pair lists; one CTA per camera row, shared-memory
 * accumulators, deterministic per-warp slot ownership */
int bamg_schur_numeric_rows(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const int32_t* pt_ptr,
                            const int32_t* obs_cam_pm, const int32_t* obs_pt_pm, const double* J, const double* A,
                            const int32_t* S_ptr, const int32_t* S_col, const int32_t* dpos, const int32_t* up_off,
                            const int32_t* up_tpos, int32_t nc, double* S, void* stream);
/* diagonal blocks (and, rhs != NULL, the right-hand side -g - sum F^T q in the same pass)
 * plus the upper off-diagonal blocks from the pair lists */
int bamg_schur_numeric(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J,
                       const double* A, const int32_t* dpos, int32_t nc, const int32_t* up_blk, const int32_t* up_tpos,
                       int32_t n_up, const int32_t* blk_pair_ptr, const int32_t* pair_a, const int32_t* pair_b,
                       const double* qo, const double* g_cam, double* rhs, double* S, void* stream);

/* point-chunk phased assembly (same sums as bamg_schur_numeric, chunk-then-point order):
 * chunk_pairs sorts the point pairs by (chunk, S block) -- chunks of consecutive points in
 * (first camera, point) order holding ~chunk_records observations each -- into pair_a /
 * pair_b / sorted_key (n_pairs each); out_host = [n_segments, n_chunks, blk_bits,
 * chunk_records used]. chunk_work builds the work list (int4 per item, capacity
 * n_segments + 10 n_chunks); out_host[0] = items. numeric_chunked runs the diagonal pass
 * and the work list; done = nnz scratch words. */
int bamg_schur_chunk_pairs(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm, const int32_t* S_ptr,
                           const int32_t* S_col, int32_t nc, int32_t npt, int64_t nnz, int64_t k,
                           const int32_t* pair_off, int64_t n_pairs, int64_t chunk_records, int32_t* pair_a,
                           int32_t* pair_b, uint32_t* sorted_key, int64_t* out_host, void* stream);
int bamg_schur_chunk_work(bamg_ctx* ctx, const int32_t* S_ptr, const int32_t* S_col, int32_t nc,
                          const uint32_t* sorted_key, int64_t n_pairs, int32_t n_seg, int32_t n_chunks,
                          int32_t blk_bits, int32_t group_rows, int32_t* work, int64_t work_cap, int64_t* out_host,
                          void* stream);
int bamg_schur_numeric_chunked(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J,
                               const double* A, const int32_t* dpos, int32_t nc, const int32_t* work, int32_t n_work,
                               const int32_t* pair_a, const int32_t* pair_b, uint32_t* done, int64_t nnz,
                               const double* qo, const double* g_cam, double* rhs, double* S, void* stream);

/* ---- BSR kernels: blockmat.py:295-299 (matvec), 91-129 (block-diagonal), 270-282 ---- */
int bamg_bsr_spmv(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col, const double* blocks,
                  const double* x, double* y, int32_t nbr, double* dot_out_dev, void* stream);
int bamg_bsr_residual(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col, const double* blocks,
                      const double* x, const double* b, double* r, int32_t nbr, void* stream);
int bamg_block_chol_inv(bamg_ctx* ctx, const double* M, int32_t n, int32_t bs, double* L, double* inv,
                        int32_t* bad_min_dev, void* stream);
int bamg_blockdiag_apply(bamg_ctx* ctx, const double* M, const double* x, int32_t n, int32_t bs, double* y,
                         void* stream);
int bamg_diag_blocks(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks, int32_t nbr,
                     int32_t bs, double* D, void* stream);

/* ---- generic block-sparse API (blockmat.py:152-360; the path's own operators use the
 *      dedicated kernels above) ---- */
/* blockmat.py:186-191 checks: flags_dev[0] = 1 when indptr decreases, flags_dev[1] = 1 when a
 * column index lies outside [0, nbc) */
int bamg_bsr_validate(bamg_ctx* ctx, const int32_t* ptr, int32_t nbr, const int32_t* col, int64_t nnz, int32_t nbc,
                      int32_t* flags_dev, void* stream);
/* blockmat.py:195-230 from_triplets. Step 1: stable (row, col) order (np.lexsort) -> perm (n),
 * seg (n: distinct entries before each sorted position); count_dev[0] = distinct entries,
 * count_dev[1] = 1 when a row / column index is out of range. Step 2: duplicates summed in
 * input order (np.add.reduceat), CSR out (ptr nbr+1, col nu, blocks nu*bsz). */
int bamg_triplets_order(bamg_ctx* ctx, const int64_t* rows, const int64_t* cols, int64_t n, int32_t nbr, int32_t nbc,
                        int32_t* perm, int32_t* seg, int32_t* count_dev, void* stream);
int bamg_triplets_reduce(bamg_ctx* ctx, const int64_t* rows, const int64_t* cols, const double* blocks, int64_t n,
                         int32_t bsz, const int32_t* perm, const int32_t* seg, int64_t nu, int32_t nbr, int32_t* ptr,
                         int32_t* col_out, double* blocks_out, void* stream);
/* blockmat.py:295-306 matvec of any block shape (rbs x cbs), scipy bsr_matvec summation order */
int bamg_bsr_matvec_gen(bamg_ctx* ctx, int32_t rbs, int32_t cbs, const int32_t* ptr, const int32_t* col,
                        const double* blocks, const double* x, int32_t nbr, double* y, void* stream);
/* blockmat.py:321-334 scale_block_columns: out_n = blocks_n @ col_blocks[col_n] (rbs x cbs @ cbs x k) */
int bamg_bsr_scale_cols(bamg_ctx* ctx, const double* blocks, const double* col_blocks, const int32_t* col,
                        int64_t nnz, int32_t rbs, int32_t cbs, int32_t k, double* out, void* stream);
/* blockmat.py:337-360 multiply / triple_product: block SpGEMM with scipy csr_matmat's summation
 * order and zero-drop. create -> *nu_host candidate blocks; numeric -> *nkeep_host kept blocks;
 * finish -> CSR (ptr a_nbr+1, col nkeep, blocks nkeep*rbs*cbs). */
typedef struct bamg_spgemm bamg_spgemm;
bamg_spgemm* bamg_spgemm_create(bamg_ctx* ctx, const int32_t* a_ptr, const int32_t* a_col, int32_t a_nbr,
                                int64_t a_nnz, const int32_t* b_ptr, const int32_t* b_col, int32_t b_nbc,
                                int64_t* nu_host, void* stream);
int bamg_spgemm_numeric(bamg_ctx* ctx, bamg_spgemm* sp, const double* a_blocks, int32_t rbs, int32_t kbs,
                        const double* b_blocks, int32_t cbs, int64_t* nkeep_host, void* stream);
int bamg_spgemm_finish(bamg_ctx* ctx, bamg_spgemm* sp, int32_t* ptr, int32_t* col, double* blocks, void* stream);
void bamg_spgemm_destroy(bamg_spgemm* sp);

/* ---- multigrid setup: multigrid.py:83-98, 127-176, 179-237, 409-471; problem.py:332-352 ---- */
int bamg_operator_strength(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks, int32_t n,
                           int64_t nnz, int32_t bs, double* nrm_work, double* dnorm_work, int32_t* G_ptr,
                           int32_t* G_col, double* G_val, int32_t* flags_dev, void* stream);
/* n_agg_dev[0] = number of aggregates, n_agg_dev[1] = largest aggregate size;
 * nnz_cap: capacity of G_col / G_val (>= G_ptr[n]; no size readback needed) */
int bamg_aggregate(bamg_ctx* ctx, const int32_t* G_ptr, const int32_t* G_col, const double* G_val, int32_t n,
                   int32_t max_size, int32_t* agg, int32_t* size_work, int32_t* n_agg_dev, int64_t nnz_cap,
                   void* stream);
int bamg_aggregate_members(bamg_ctx* ctx, const int32_t* agg, int32_t n, int32_t n_agg, int32_t* agg_ptr,
                           int32_t* members, void* stream);
int bamg_gauge_nullspace(bamg_ctx* ctx, const double* cams, int32_t nc, double* K, void* stream);
int bamg_prolongation_qr(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members, const double* K,
                         int32_t n_agg, int32_t bs, int32_t max_members, double* Pblocks, double* Kc, int32_t* info,
                         int32_t* padded_cnt, void* stream);
int bamg_galerkin_pattern(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members, const int32_t* ptr,
                          const int32_t* col, const int32_t* agg, int32_t n_agg, int32_t* Cptr_or_counts,
                          int32_t* Ccol, void* stream);
int bamg_galerkin_map(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const int32_t* agg, int32_t n,
                      int64_t nnz_fine, const int32_t* Cptr, const int32_t* Ccol, int64_t nnz_coarse,
                      int32_t* fine_sorted, int32_t* cblk_ptr, int32_t* fine_row, void* stream);
/* A_{l+1} = sym(P^T A_l P) (multigrid.py:409, 444-471): only the upper coarse blocks are
 * multiplied out; each is stored with its transpose at the mirror position (diagonal
 * blocks: 0.5 (C + C^T)), then the padded-dof patch. nnz_fine = fine blocks in the map. */
int bamg_galerkin_numeric(bamg_ctx* ctx, int32_t bs, const int32_t* cblk_ptr, const int32_t* fine_sorted,
                          const int32_t* fine_row, const int32_t* col, const double* blocks, const double* P,
                          int64_t nnz_fine, int32_t n_agg, const int32_t* Cptr, const int32_t* Ccol,
                          int64_t nnz_coarse, const int32_t* padded_cnt, double* out, void* stream);
/* coarsest direct solve: multigrid.py:431-440 (cho_factor) / 477-478 (cho_solve) */
int bamg_coarse_factor(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks, int32_t nbr,
                       int32_t bs, double* dense, double* work, double* inv, int32_t* flag_dev, void* stream);
int bamg_dense_gemv(bamg_ctx* ctx, const double* M, const double* x, int32_t n, double* y, void* stream);

/* ---- smoother / V-cycle / PCG: multigrid.py:308-328, 474-483; solver.py:70-128 ---- */
int bamg_cheb_step(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col, const double* blocks,
                   const double* x_in, const double* b, const double* Dinv, double* d, double* x_out, int32_t nbr,
                   double c1, double c2, int32_t divide, void* stream);
int bamg_prolong(bamg_ctx* ctx, const int32_t* agg, const double* P, const double* xc, int32_t nf, int32_t bs,
                 double* y, int32_t accumulate, void* stream);
int bamg_restrict(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members, const double* P, const double* r,
                  int32_t nagg, int32_t bs, double* bc, void* stream);
int bamg_pcg_update(bamg_ctx* ctx, double* x, double* r, const double* p, const double* ap, double alpha,
                    int64_t n, double* rr_dev, void* stream);
int bamg_xpby(bamg_ctx* ctx, const double* z, double beta, double* p, int64_t n, void* stream);
/* multigrid.py:281-284: largest eigenvalue of the Lanczos tridiagonal (host arrays) */
double bamg_tridiag_max_eig(const double* a_host, const double* b_host, int32_t n);

/* ---- driver helpers: rotation.py:124-137 canonicalize (solver.py:290, problem.py:106) ---- */
int bamg_canonicalize(bamg_ctx* ctx, double* cams, int32_t n, int32_t stride, void* stream);
/* solver.py:276-301 LM trial decision on the device: t_dev = [rhs.dc, dc.S dc, g_p.C^-1 g_p,
 * dc.dc, dp.dp, f, f_new, radius] (device scalars), n_behind_dev = the candidate's behind-camera
 * count. Computes decrease (schur.py:176-188), rho, accepted = rho > min_rho; on accept
 * copies the candidate into (cams, pts) and canonicalises the rotations. out_dev =
 * [rho, accepted, decrease, step_norm, f_new, radius'] (6 doubles) with the trust-region
 * update of solver.py:134-149 applied to the radius -- one readback per LM trial. */
int bamg_lm_trial(bamg_ctx* ctx, const double* t_dev, const int32_t* n_behind_dev, double min_rho, double* cams,
                  const double* cand_cams, int32_t nc, double* pts, const double* cand_pts, int32_t npt,
                  double* out_dev, void* stream);
/* number of library kernel launches so far (benchmark accounting) */
int64_t bamg_launch_count(void);

/* ---- problem files: balio.py:25-97 (host side, multi-threaded; HOST pointers) ----
 * read: header counts first, then the caller sizes the arrays and reads. Return 0,
 * BAMG_ERR_FORMAT with *err_line (1-based) and the reference's message, or <0 on an
 * I/O failure (message in err_msg). n_threads <= 0: all hardware threads. */
int bamg_bal_read_header(const char* path, int64_t* counts3, int64_t* err_line, char* err_msg, size_t err_len);
int bamg_bal_read(const char* path, int64_t n_cam, int64_t n_pt, int64_t n_obs, int64_t* cam_index,
                  int64_t* pt_index, double* pixels, double* cams, double* pts, int32_t n_threads,
                  int64_t* err_line, char* err_msg, size_t err_len);
/* write: "%d %d %.17g %.17g" observation lines, one %.17g scalar per line (bit-exact round trip) */
int bamg_bal_write(const char* path, int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_index,
                   const int64_t* pt_index, const double* pixels, const double* cams, const double* pts,
                   int32_t n_threads);

/* ---- visibility block-Jacobi (precond.py:59-144) ----
 * Clusters c = 0..ncl-1 (aggregation with cap 100, multigrid.py:127-176), members
 * mem[cptr[c]..cptr[c+1]) ascending, agg[camera] = cluster. Each cluster's principal
 * submatrix of S (dim[c] = 9 |members|, row-major at off[c] doubles) is assembled
 * from the explicit S (precond.py:96-111), Cholesky-factored (flags[c] = 1 when not
 * positive definite: IndefiniteBlockError(c), precond.py:139-143) and inverted;
 * the apply replaces the per-cluster cho_solve of VisibilityJacobi.apply (69-78). */
int bamg_vj_assemble(bamg_ctx* ctx, const int32_t* S_ptr, const int32_t* S_col, const double* S_blocks, int32_t nc,
                     const int32_t* agg, const int32_t* cptr, const int32_t* mem, const int64_t* off,
                     const int32_t* dim, double* dense, int64_t total, void* stream);
int bamg_vj_factor(bamg_ctx* ctx, int32_t ncl, int32_t dim_max, const int64_t* off, const int32_t* dim, double* work,
                   double* tmp, double* inv, int32_t* flags, void* stream);
typedef struct bamg_vj bamg_vj;
bamg_vj* bamg_vj_create(int32_t ncl, int32_t dim_max, const int64_t* off, const int32_t* dim, const int32_t* cptr,
                        const int32_t* mem, const double* inv);
void bamg_vj_destroy(bamg_vj* vj);
int bamg_vj_apply(bamg_ctx* ctx, const bamg_vj* vj, const double* r, double* z, void* stream);

/* ---- native solve-phase runtime ----
 * A multigrid plan holds per-level operators (device pointers owned by the caller)
 * and its own work vectors; the V-cycle (mgcycle, multigrid.py:474-483, with the
 * Chebyshev smoother of multigrid.py:308-328) is recorded once as a CUDA graph. */
typedef struct bamg_mg bamg_mg;
bamg_mg* bamg_mg_create(int32_t n_levels);
void bamg_mg_destroy(bamg_mg* mg);
int bamg_mg_set_level(bamg_mg* mg, int32_t level, int32_t bs, int32_t nbr, const int32_t* ptr, const int32_t* col,
                      const double* blocks, const double* Dinv, double lower, double upper, int32_t iterations,
                      const double* P, const int32_t* agg, const int32_t* agg_ptr, const int32_t* members,
                      int32_t n_agg, const double* coarse_inv);
/* Symmetric half-storage view of the explicit S (9x9 blocks): the solve phase
 * streams only the upper blocks (positions dpos[i]..ptr[i+1]-1) and forms the lower
 * half from their transposes (S_ji == S_ij^T exactly, schur.py:143-144). Built from
 * the upper-block list of the Schur symbolic phase; owns its mirror map and the
 * transposed-product buffer (9 nnzb doubles). Replaces bsr_matvec on S inside
 * SchurSystem.matvec / the V-cycle (blockmat.py:295-299). */
typedef struct bamg_symop bamg_symop;
bamg_symop* bamg_symop_create(int32_t nbr, const int32_t* ptr, const int32_t* col, const int32_t* dpos,
                              const int32_t* up_blk, const int32_t* up_tpos, int32_t n_up, int64_t nnzb, void* stream);
/* the same view for any exactly symmetric BSR pattern (bs 9 or 16: the Galerkin
 * coarse operators, multigrid.py:444-455 symmetrises them), diagonal slots and
 * mirror positions derived from (ptr, col) */
bamg_symop* bamg_symop_create_pattern(int32_t bs, int32_t nbr, const int32_t* ptr, const int32_t* col, int64_t nnzb,
                                      void* stream);
void bamg_symop_destroy(bamg_symop* sym);
/* pass-1 work units (row chunks) of the view */
int32_t bamg_symop_chunks(const bamg_symop* sym);
int bamg_symop_spmv(bamg_ctx* ctx, const bamg_symop* sym, const double* blocks, const double* x, double* y,
                    double* dot_out_dev, void* stream);
/* r = b - S x, and the fused Chebyshev step of bamg_cheb_step, through the half-storage view */
int bamg_symop_residual(bamg_ctx* ctx, const bamg_symop* sym, const double* blocks, const double* x,
                        const double* b, double* r, void* stream);
int bamg_symop_cheb_step(bamg_ctx* ctx, const bamg_symop* sym, const double* blocks, const double* x_in,
                         const double* b, const double* Dinv, double* d, double* x_out, double c1, double c2,
                         int32_t divide, void* stream);
int bamg_mg_set_symmetric(bamg_mg* mg, int32_t level, const bamg_symop* sym);
/* coarse V-cycle tail as one persistent cooperative kernel: levels whose 16x16
 * operator is at most max_mb MB (0 disables; -1 = BAMG_VTAIL_MB, default 0) */
int bamg_mg_set_tail(bamg_mg* m, int32_t max_mb);
int bamg_mg_use_graph(bamg_mg* mg, int32_t on);
/* arena + graph ahead of the first bamg_mg_apply (optional; apply prepares lazily) */
int bamg_mg_prepare(bamg_ctx* ctx, bamg_mg* mg, void* stream);
int bamg_mg_apply(bamg_ctx* ctx, bamg_mg* mg, const double* r, double* z, void* stream);
/* how the prepared plan runs level l's products (measurement only): 0 half-storage
 * pair, 1 one-CTA-per-row full storage, 2 chunked full storage, 3 warp-per-row full
 * storage, 4 coarsest (dense inverse); -1 before the first application */
int32_t bamg_mg_level_kind(const bamg_mg* mg, int32_t level);
/* solver.py:70-128 pcg with a BSR operator and the MG plan (or block-Jacobi inverse
 * blocks when mg == NULL); one host synchronisation per iteration. err codes:
 * 1 PreconditionerNotSPD, 2/3/4/5 CgDivergence (operator non-finite / curvature /
 * residual non-finite / preconditioner non-finite). */
/* optional: build the PCG graph of a later bamg_pcg_run with the same arguments now (host
 * capture / re-target overlaps device work in flight) */
int bamg_pcg_prepare(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs, int32_t nbr,
                     const int32_t* ptr, const int32_t* col, const double* blocks, const double* b, double* x,
                     double tau, int32_t max_it, double rtol, double* work, const bamg_symop* sym, void* stream);
int bamg_pcg_run(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs, int32_t nbr,
                 const int32_t* ptr,
                 const int32_t* col, const double* blocks, const double* b, double* x, double tau, int32_t max_it,
                 double rtol, double* work, int32_t* iterations_out, int32_t* reason_out, double* rel_out,
                 double* q_hist, int32_t* err_out, double* err_value_out, int32_t* err_iter_out,
                 const bamg_symop* sym, void* stream);
/* multigrid.py:243-284 estimate_lambda_max for a BSR operator; work: (steps+5)*n doubles */
int bamg_lanczos_lmax(bamg_ctx* ctx, int32_t bs, int32_t nbr, const int32_t* ptr, const int32_t* col,
                      const double* blocks, const double* D, const double* Dinv, const double* v0, int32_t steps,
                      double* work, double* lambda_out, int32_t* status, const bamg_symop* sym,
                      double* ab_out_dev, void* stream);
/* ab_out_dev != NULL: no readback -- the 16 scalars [alpha_0..7 | beta^2_0..7] land in
 * ab_out_dev and bamg_lanczos_finish (host) replays the break rule and the Ritz max
 * later, so several levels share one readback */
int bamg_lanczos_finish(const double* ab_host, int32_t steps, double* lambda_out, int32_t* status);

/* ---- device-side synthetic scenes, BASELINE configs 3-5 ----
 * The model of the reference's host generator (synth.py:92-558: look-at camera frames,
 * visibility draw, pixel noise, centre-preserving start perturbation) with the
 * distributions of SURVEY App. C (scenes.py is the numpy statement used for the goldens).
 * kind: 3 city, 4 large, 5 loop. params_host (8 doubles, host memory): [side, n_clusters,
 * cam_sigma, pt_sigma, z_max, lam, radius (= grid cell), bridge_frac]. Counter-based RNG:
 * every draw is a function of (seed, stream, index).
 * layout: cam_centre (nc,3), cam_rt (nc,24: R, t, R0, t0), cam_truth / cam_init (nc,9),
 *   cam_cell (nc) grid cell of each camera, pts_true / pts_init (npts,3), n_pick (npts)
 *   requested cameras, aux (npts,2) loop run placement.
 * visibility: cell_ptr / cell_cams = cameras grouped by cell (kinds 3, 4); sel
 *   (npts x 32) the surviving cameras of each point sorted by camera, cnt (npts; 0 when
 *   fewer than two survive), cam_used (nc) / pt_used (npts) 0/1 flags, info[0] = points
 *   whose in-radius candidates overflowed the 2048-entry cache (must be 0).
 * emit: obs_off = exclusive scan of cnt, cam_map / pt_map = exclusive scans of the used
 *   flags; writes the compacted problem arrays (observations point-major). */
int bamg_scene_grid_cells(int32_t kind, int32_t nc, int64_t npts, const double* params_host);
int bamg_scene_layout(bamg_ctx* ctx, int32_t kind, int64_t seed, int32_t nc, int64_t npts,
                      const double* params_host, double* cam_centre, double* cam_rt, double* cam_truth,
                      double* cam_init, uint32_t* cam_cell, double* pts_true, double* pts_init,
                      int32_t* n_pick, int32_t* aux, void* stream);
int bamg_scene_visibility(bamg_ctx* ctx, int32_t kind, int64_t seed, int32_t nc, int64_t npts,
                          const double* params_host, int32_t k_nn, const double* cam_centre,
                          const double* cam_rt, const double* pts_true, const double* pts_init,
                          const int32_t* n_pick, const int32_t* aux, const int32_t* cell_ptr,
                          const uint32_t* cell_cams, int32_t* sel, int32_t* cnt, int32_t* cam_used,
                          int32_t* pt_used, int32_t* info, void* stream);
int bamg_scene_emit(bamg_ctx* ctx, int64_t seed, int32_t nc, int64_t npts, const int32_t* cnt,
                    const int32_t* obs_off, const int32_t* sel, const int32_t* cam_used,
                    const int32_t* cam_map, const int32_t* pt_map, const double* cam_rt,
                    const double* cam_truth, const double* cam_init, const double* pts_true,
                    const double* pts_init, int64_t* cam_index, int64_t* pt_index, double* pixels,
                    double* out_cam_truth, double* out_cam_init, double* out_pts_true,
                    double* out_pts_init, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BAMG_B200_H */
