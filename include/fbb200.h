/*
 * fbb200.h — C ABI of the B200-native sum-factorized operator path.
 *
 * This is the drop-in boundary for the hot path of the flowbench reference
 * (arXiv 1910.03032): the matrix-free operator action (mass, stiffness,
 * Helmholtz, vector Laplacian, gradient, divergence) applied inside the
 * Krylov loops, plus the Krylov vector kernels and the LOR V-cycle pieces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "_dev" pointers are CUDA device
 *    pointers; "_host" pointers are host memory read during the call only.
 *  - Every function returns an int status: FB_OK (0) or one of the FB_ERR_*
 *    codes below, with a thread-local message from fb_last_error().  The
 *    Python layer maps FB_ERR_ARG to ValueError (the reference raises
 *    ValueError for shape / kind mismatches, mfop.py:192-193, 253-254, 452),
 *    FB_ERR_OOM to MemoryError and everything else to RuntimeError.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - Objects own their device data (maps, transposed maps, factors, 1D
 *    matrices); apply calls allocate nothing.
 *  - Numbering, layouts and index conventions are those of the reference:
 *    local DoF l = i0 + n*i1 + n^2*i2 (fespace.py:23-28), quadrature point
 *    q0 + nq*q1 + nq^2*q2 (mesh.py:204-213), vector fields struct-of-arrays
 *    (fespace.py:10-12).
 */
#ifndef FBB200_H
#define FBB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_OK 0
#define FB_ERR_ARG 1          /* bad shape / argument / kind        */
#define FB_ERR_CUDA 2         /* CUDA runtime error                 */
#define FB_ERR_OOM 3          /* device allocation failed           */
#define FB_ERR_UNSUPPORTED 4  /* configuration not built            */

/* Operator kinds (mfop.setup kinds, mfop.py:436-452). */
#define FB_MASS 0
#define FB_STIFFNESS 1
#define FB_HELMHOLTZ 2
#define FB_GRADIENT 3
#define FB_DIVERGENCE 4
#define FB_CONVECTION 5  /* nonlinear (u . grad) u load, mfop.py:322-358 */
#define FB_CURLCURL 6    /* weak rotational viscous term, mfop.py:361-413 */

typedef struct fb_restriction fb_restriction;
typedef struct fb_operator fb_operator;
typedef struct fb_csr fb_csr;
typedef struct fb_transfer fb_transfer;
typedef struct fb_trisolve fb_trisolve;
typedef struct fb_blockilu fb_blockilu;

const char* fb_last_error(void);
int fb_abi_version(void);
/* Number of kernel launches issued by this library since load (evidence
 * counter used by bench.py's gpu_launches). */
int64_t fb_launch_count(void);

/* ------------------------------------------------------------------ */
/* Element restriction: replaces FESpace.gather / FESpace.scatter_add   */
/* (fespace.py:282-292).                                                */
/* ------------------------------------------------------------------ */

/* element_dofs_host: (ne, (p+1)^dim) int64, the reference's
 * FESpace.element_dofs (fespace.py:71-217).  Builds the int32 L->E map, the
 * transposed CSR used by the deterministic E->L sum (ascending flat E
 * index, bitwise equal to np.bincount), and the split between element-
 * interior DoFs (written directly by the operator kernels) and shared DoFs. */
int fb_restriction_create(int dim, int p, int64_t ne, int64_t ndofs,
                          const int64_t* element_dofs_host, fb_restriction** out);
void fb_restriction_destroy(fb_restriction* r);
int64_t fb_restriction_ndofs(const fb_restriction* r);
/* xe_dev = x_dev[element_dofs]   (fespace.py:282-284) */
int fb_restriction_gather(const fb_restriction* r, const double* x_dev, double* xe_dev,
                          void* stream);
/* y_dev = bincount(element_dofs, xe)   (fespace.py:286-292) */
int fb_restriction_scatter_add(const fb_restriction* r, const double* xe_dev, double* y_dev,
                               void* stream);

/* ------------------------------------------------------------------ */
/* Sum-factorized operators (mfop.py:169-319).                          */
/* ------------------------------------------------------------------ */

/* kind: FB_MASS | FB_STIFFNESS | FB_HELMHOLTZ  (square operators on rv,
 *       vdim components sharing factors, _SquareOperator mfop.py:169-244)
 *       FB_GRADIENT | FB_DIVERGENCE  (rv = velocity restriction (scalar
 *       numbering), rp = pressure restriction, vdim = dim; mfop.py:247-319)
 * nq1, points_host: 1D rule size and points (geom.rule.points).
 * B_host/D_host: (nq1, nv) basis values/derivatives of the (velocity) space
 *       at the rule points (basis.py:122-156); Bp/Dp: (nq1, np) for the
 *       pressure space (NULL for square kinds).
 * wdet_host: (ne, nq1^dim) mass factor incl. any c (mfop.py:129-130, 234), or NULL
 * stiff_host: (ne, nq1^dim, dim(dim+1)/2) packed symmetric factor (mfop.py:133-142), or NULL
 * grad_host:  (ne, nq1^dim, dim, dim) (mfop.py:145-152), or NULL
 * All factor arrays are in the reference's AoS layout; they are re-laid
 * out element-blocked on the device. */
int fb_operator_create(int kind, const fb_restriction* rv, const fb_restriction* rp,
                       int vdim, int nq1, const double* points_host,
                       const double* B_host, const double* D_host,
                       const double* Bp_host, const double* Dp_host,
                       const double* wdet_host, const double* stiff_host,
                       const double* grad_host, fb_operator** out);
/* Same operator, with the quadrature-point factors computed on the device
 * from the element corners (ne, 2^dim, dim) (compute_geometric_factors,
 * mesh.py:216-267, then mfop.py:129-152): weights = 1D rule weights;
 * c = Helmholtz mass coefficient, nu = viscosity (mfop.py:211-244). */
int fb_operator_create_geom(int kind, const fb_restriction* rv, const fb_restriction* rp,
                            int vdim, int nq1, const double* points_host,
                            const double* weights_host, const double* B_host,
                            const double* D_host, const double* Bp_host, const double* Dp_host,
                            const double* corners_host, double c, double nu,
                            fb_operator** out);
/* Select one of the compiled launch shapes (0..7) of the fused kernel for
 * degree p, or -1 to restore the tuned default; used by tools/tune_fast.py
 * and the multi-batch parity tests. */
int fb_set_fast_config(int p, int variant);
/* Shape of the last persistent fused-kernel launch on the calling thread:
 * CTAs, element batches and elements per batch (each CTA walks
 * nbatch / grid batches).  Test/diagnostic query. */
int fb_last_fast_launch(int* grid, int* nbatch, int* elements_per_batch);
/* Diagnostics (tools/pass_cost.py): skip the arithmetic of the fused
 * kernel's passes P1..P9 whose bits are set in `mask` (results invalid);
 * 0 restores normal operation. */
int fb_set_fast_skip(int mask);
/* Element-blocked factors (ne, K, nq1^dim) back to host, for verification. */
int64_t fb_operator_factor_count(const fb_operator* op);
int fb_operator_factors(const fb_operator* op, double* host_out, int64_t count);
void fb_operator_destroy(fb_operator* op);
/* y = A x.  Square kinds: x, y of length vdim*ndofs.  Gradient: x pressure,
 * y velocity.  Divergence: x velocity, y pressure. */
int fb_operator_apply(const fb_operator* op, const double* x_dev, double* y_dev, void* stream);
/* Fused path only: part 1 = element kernel (interior DoFs to y, shared
 * contributions to the operator's buffer), part 2 = the E->L sum of the
 * shared DoFs, part 0 = both (== fb_operator_apply).  For kernel timing. */
int fb_operator_apply_part(const fb_operator* op, const double* x_dev, double* y_dev, int part,
                           void* stream);
/* Gradient only: y = G^T x (GradientOperator.apply_transpose, mfop.py:277-288). */
int fb_operator_apply_transpose(const fb_operator* op, const double* x_dev, double* y_dev,
                                void* stream);
/* Bytes of device memory the operator owns (factors + matrices). */
int64_t fb_operator_device_bytes(const fb_operator* op);
/* 1 if the fused sm_100a kernel serves this square operator, 2 if the fused
 * mixed-degree kernel serves this gradient / divergence, 0 for the general kernel. */
int fb_operator_fast_path(const fb_operator* op);

/* ConstrainedOperator.apply (mfop.py:428-433) around any operator apply:
 * xi = x; xi[dofs] = 0; y = A xi; y[dofs] = x[dofs].  `work_dev` holds
 * a length-n scratch vector. */
int fb_mask_copy_zero(const double* x_dev, double* xi_dev, int64_t n, const int64_t* dofs_dev,
                      int64_t ndofs, void* stream);
int fb_mask_restore(const double* x_dev, double* y_dev, const int64_t* dofs_dev, int64_t ndofs,
                    void* stream);

/* Reference DoF numbering (fespace.py:71-217) on the host, for a mesh given
 * by its element -> vertex-class table (ne, 2^dim).  element_dofs_out:
 * (ne, (p+1)^dim).  Returns ndofs_scalar, or minus a status code. */
int64_t fb_number_dofs_host(int dim, int p, int64_t ne, int64_t nv, const int64_t* elements,
                            int64_t* element_dofs_out, int64_t* num_edges, int64_t* num_faces);

/* ------------------------------------------------------------------ */
/* Krylov vector kernels (solvers.py:108-254).  Deterministic: partial  */
/* sums over fixed 4096-entry chunks, then a fixed-order second pass.   */
/* ------------------------------------------------------------------ */
/* partial_dev must hold fb_dot_partials(n) doubles; result_dev one. */
int64_t fb_dot_partials(int64_t n);
int fb_dot(int64_t n, const double* x_dev, const double* y_dev, double* partial_dev,
           double* result_dev, void* stream);
/* y = a*x + b*y  (a, b host scalars) */
int fb_axpby(int64_t n, double a, const double* x_dev, double b, double* y_dev, void* stream);
/* Fused PCG update (reference solvers.py:141-150 `alpha = rz / pAp;
 * x += alpha * p; r -= alpha * Ap`): alpha_out[0] = rz/pAp (0 if pAp <= 0),
 * x += alpha p and, if update_r, r -= alpha Ap in one pass; numpy rounding. */
int fb_cg_update(int64_t n, const double* rz_dev, const double* pAp_dev, double* alpha_out_dev,
                 const double* p_dev, const double* Ap_dev, double* x_dev, double* r_dev,
                 int update_r, void* stream);
/* y = a_dev[0]*x + y, scalar read on device (alpha = rz/pAp, kept on device) */
int fb_axpy_dev(int64_t n, const double* a_dev, int sign, const double* x_dev, double* y_dev,
                void* stream);
/* scalar ops on device: out = num/den */
int fb_scalar_div(const double* num_dev, const double* den_dev, double* out_dev, void* stream);
/* p = z + beta*p with beta = num/den read on device */
int fb_xpby_ratio(int64_t n, const double* z_dev, const double* num_dev, const double* den_dev,
                  double* p_dev, void* stream);
/* y = a * x (a host scalar) */
int fb_scale(int64_t n, double a, const double* x_dev, double* y_dev, void* stream);
/* y = x / s (s host scalar; the reference's `r / beta`, fgmres) */
int fb_div_scalar(int64_t n, const double* x_dev, double s, double* y_dev, void* stream);
/* y = x - num_dev[0] / den  (mean deflation, solvers.py:60-64) */
int fb_shift_ratio(int64_t n, const double* x_dev, const double* num_dev, double den,
                   double* y_dev, void* stream);
/* out = den > 0 ? num / den : 0  (CG step length with the pAp <= 0 guard) */
int fb_safe_div(const double* num_dev, const double* den_dev, double* out_dev, void* stream);
/* y = d .* x */
int fb_vmul(int64_t n, const double* d_dev, const double* x_dev, double* y_dev, void* stream);

/* ------------------------------------------------------------------ */
/* Sparse pieces of the LOR V-cycle (solvers.py:269-392, lor.py:61-123) */
/* ------------------------------------------------------------------ */
/* CSR matrix on the device (int64 row offsets, int32 column indices, fp64
 * values), copied from host int64 CSR arrays (scipy.sparse.csr_matrix). */
int fb_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* indptr_host,
                  const int64_t* indices_host, const double* data_host, fb_csr** out);
void fb_csr_destroy(fb_csr* A);
/* y = A x, rows summed sequentially in index order (scipy csr_matvec order) */
int fb_csr_spmv(const fb_csr* A, const double* x_dev, double* y_dev, void* stream);
/* y = b - A x */
int fb_csr_residual(const fb_csr* A, const double* b_dev, const double* x_dev, double* y_dev,
                    void* stream);
/* y_j = b_j - A x_j (b NULL: y_j = A x_j) for nv = 1..4 vectors stored at a
 * common stride (the components of a vector field sharing one scalar level
 * matrix): each entry is read once; per vector bitwise fb_csr_residual. */
int fb_csr_residual_multi(const fb_csr* A, int nv, const double* b_dev, const double* x_dev,
                          double* y_dev, int64_t stride, void* stream);
/* Sparse triangular solve T x = b (lower=1: forward, 0: backward; unit_diag
 * ignores/omits the diagonal).  Sync-free: one launch per solve. */
int fb_trisolve_create(int64_t n, const int64_t* indptr_host, const int64_t* indices_host,
                       const double* data_host, int lower, int unit_diag, fb_trisolve** out);
void fb_trisolve_destroy(fb_trisolve* T);
int fb_trisolve_solve(const fb_trisolve* T, const double* b_dev, double* x_dev, void* stream);
/* Number of dependency levels of the triangular matrix. */
int fb_trisolve_levels(const fb_trisolve* T);
/* Solve strategy for all triangular solves: 0 = sync-free single launch
 * (poll backoff in ns), 1 = level-scheduled kernels replayed from a CUDA graph. */
int fb_set_trisolve_mode(int mode, int backoff_ns);
/* dst[i] = src[idx[i]] (scatter=0) or dst[idx[i]] = src[i] (scatter=1) */
int fb_permute(int64_t n, const int* idx_dev, const double* src_dev, double* dst_dev, int scatter,
               void* stream);
/* Block-Jacobi ILU(0) smoother (scale mode of the LOR V-cycle, SURVEY
 * 8(e')): F = block-diagonal ILU(0) factor in block-major numbering (strict
 * lower = L with unit diagonal, upper incl. diagonal = U), block_ptr =
 * (nblocks+1) row offsets, new2old = new -> original index.  apply computes
 * out = (LU)^-1 r (transpose=0) or (LU)^-T r (transpose=1) in the original
 * numbering with one CTA per block, level-scheduled in shared memory. */
int fb_blockilu_create(int64_t n, int nblocks, const int64_t* block_ptr_host,
                       const int64_t* new2old_host, const int64_t* indptr_host,
                       const int64_t* indices_host, const double* data_host, fb_blockilu** out);
void fb_blockilu_destroy(fb_blockilu* B);
/* Sizes of the factor: rows, strict-lower / strict-upper entries (the
 * V-cycle's algorithmic bytes), padded row width of the sweeps (0: CSR). */
int fb_blockilu_info(const fb_blockilu* B, int64_t* n, int64_t* nnz_lower, int64_t* nnz_upper,
                     int* ell_width);
int fb_blockilu_apply(const fb_blockilu* B, int transpose, const double* r_dev, double* out_dev,
                      void* stream);
/* Sweep the factor runs: 0 = CSR level loop, 1 = ELL, 2 = level-packed
 * TMA ring (fb_set_blockilu_packed). */
int fb_blockilu_sweep_kind(const fb_blockilu* B);
/* out += (LU)^-1 r (transpose 0) / (LU)^-T r (transpose 1): the V-cycle's
 * smoothing correction x += M^-1 (b - A x) (reference solvers.py:382) added in
 * the sweep's final store; level-packed sweeps only (sweep kind 2), else
 * FB_ERR_ARG */
int fb_blockilu_apply_add(const fb_blockilu* B, int transpose, const double* r_dev,
                          double* out_dev, void* stream);
/* y = M x for a dense row-major n x n matrix (coarse-level inverse). */
int fb_dense_mv(int64_t n, const double* M_dev, const double* x_dev, double* y_dev, void* stream);
/* LOR matrix of a degree-p space on its nodal sub-cell mesh (lor.py:61-99):
 * Q1 kind (FB_MASS / FB_STIFFNESS / FB_HELMHOLTZ) with 2-point Gauss, rows
 * in CSR with sorted columns, constrained rows/columns zeroed in-pattern with
 * a unit diagonal.  corners: (ne, 2^dim, dim); nodes: the p+1 GLL nodes.
 * Outputs are malloc'ed; release them with fb_host_free.  Returns nnz or
 * minus a status code. */
int64_t fb_lor_assemble_host(int dim, int p, int64_t ne, int64_t ndofs, const int64_t* element_dofs,
                             const double* corners, const double* nodes, int kind, double nu,
                             double c, int64_t ncons, const int64_t* constrained,
                             int64_t** indptr_out, int64_t** indices_out, double** data_out);
void fb_host_free(void* p);
/* ILU(0) in place on sorted CSR, IKJ order (kernels/numba_backend.py:64-103):
 * returns -1 on success, else the failing row. */
int64_t fb_ilu0_factor_host(int64_t n, const int64_t* indptr, const int64_t* indices,
                            double* data);

/* ------------------------------------------------------------------ */
/* Structured-box scale mode: LOR levels built on the device            */
/* (SURVEY 8(e') and 8(f) items 1-2; replaces the host setup of         */
/* lor.py:61-123, solvers.py:269-392 and numba_backend.py:64-103)       */
/* ------------------------------------------------------------------ */
/* Q1 LOR matrix of a degree-p space on a structured box of counts[3]
 * elements (numbered x fastest), assembled on the device: one row per
 * lattice point of the (counts*p+1)^3 nodal lattice, rows/columns numbered by
 * lattice_ids_dev (int32, x fastest), columns sorted.  corners_dev: (ne, 8, 3)
 * element corners; nodes: the p+1 GLL nodes (host).  constrain_boundary
 * zeroes boundary rows/columns with a unit diagonal (lor.py:84-99). */
int fb_lor_assemble_box(int p, const int64_t* counts, const double* corners_dev,
                        const double* nodes, const int* lattice_ids_dev, int kind, double nu,
                        double c, int constrain_boundary, fb_csr** out);
/* Slab-local variant (multi-GPU scale mode): constrain_faces is a bitmask of
 * the constrained box faces (1 x-, 2 x+, 4 y-, 8 y+, 16 z-, 32 z+; cut planes
 * between ranks are not constrained) plus periodic axes in bits 6-8 (64 x,
 * 128 y, 256 z: counts*p lattice points, indices wrap, mesh.py:81-96);
 * only rows with lattice id < nrows are
 * assembled (the rank's owned DoFs), columns range over ncols local ids
 * (owned + ghost planes).  nrows/ncols < 0: the whole lattice. */
int fb_lor_assemble_box_rows(int p, const int64_t* counts, const double* corners_dev,
                             const double* nodes, const int* lattice_ids_dev, int kind,
                             double nu, double c, int constrain_faces, int64_t nrows,
                             int64_t ncols, fb_csr** out);
/* Pin one DoF of a device CSR (row and column zeroed, unit diagonal; the
 * pattern must hold the diagonal): lor.constrain_matrix(A, [dof]). */
int fb_csr_pin(fb_csr* A, int64_t dof);
int fb_csr_info(const fb_csr* A, int64_t* nrows, int64_t* ncols, int64_t* nnz);
/* copy a device CSR to host arrays (indptr: nrows+1, indices/data: nnz) */
int fb_csr_download(const fb_csr* A, int64_t* indptr, int64_t* indices, double* data);
/* Block-Jacobi ILU(0) of a device CSR already numbered block-major (rows of
 * block b are block_ptr[b]..block_ptr[b+1]-1), factored and level-grouped on
 * the device; same factor and sweeps as fb_blockilu_create.  On a zero pivot
 * *fail_row >= 0 and no handle is returned (the caller falls back to Jacobi,
 * solvers.py:283-290). */
int fb_blockilu_create_csr(const fb_csr* A, int64_t nblocks, const int64_t* block_ptr_host,
                           int64_t* fail_row, fb_blockilu** out);
/* Block-ILU sweep variant for smoothers created afterwards: mode 2 = padded
 * rows (value/offset vectors, default), 1 = CSR rows with the next level's
 * loads issued early, 0 = plain CSR level loop; lanes = lanes per block (one
 * warp serves 32/lanes blocks), 0 = chosen from the block size.  Same
 * results in every mode. */
int fb_set_blockilu_pipeline(int mode, int lanes);
/* 1 (default): factors created afterwards with blocks of more than 160 rows
 * (on grids of many blocks) use the level-packed layout and the TMA-ring
 * sweep, which splits each row over 1-4 lanes (same factor; the row sums are
 * taken in a different fixed order, so results agree with the CSR / ELL
 * sweeps to rounding, and are deterministic); 0: CSR / ELL sweeps. */
int fb_set_blockilu_packed(int on);
/* Nodal interpolation between two levels of a structured box, matrix-free
 * (lor.py:102-123).  fine: map of the fine level (ne, nf^3); hmap: for each
 * fine element the coarse DoFs of its parent coarse element (ne, nc^3);
 * counts: fine element counts; W: nw weight tables (nf x nc); widx: for
 * axis a and element coordinate i, the table index (arrays of counts[0],
 * counts[1], counts[2] entries, concatenated).  Fine DoFs follow first-touch
 * ownership. */
int fb_transfer_create(const fb_restriction* fine, const fb_restriction* hmap,
                       const int64_t* counts, int nw, const double* W, const int64_t* widx,
                       fb_transfer** out);
void fb_transfer_destroy(fb_transfer* T);
/* global element coordinates of the transfer's local element (0,0,0)
 * (first-touch ownership on a slab of a larger box) */
/* Periodic axes (bitmask x 1, y 2, z 4) of a p-transfer and the global
 * element counts: the last element's local index p along a periodic axis
 * is owned by the first element (first touch). */
int fb_transfer_set_periodic(fb_transfer* T, int axes, int64_t gnx, int64_t gny, int64_t gnz);
int fb_transfer_set_origin(fb_transfer* T, int64_t x0, int64_t y0, int64_t z0);
/* y[idx[i]] += v[i] for distinct indices (slab halo partial sums) */
int fb_index_add(int64_t n, const int* idx_dev, const double* v_dev, double* y_dev, void* stream);
/* xf = P xc */
int fb_transfer_prolong(const fb_transfer* T, const double* xc_dev, double* xf_dev, void* stream);
/* xf += P xc (coarse-grid correction in place; rounding of xf = 1*(P xc) + 1*xf,
 * reference solvers.py:381 `x = x + P @ ...`) */
int fb_transfer_prolong_add(const fb_transfer* T, const double* xc_dev, double* xf_dev,
                            void* stream);
/* xc = P^T xf (deterministic) */
int fb_transfer_restrict(const fb_transfer* T, const double* xf_dev, double* xc_dev, void* stream);

/* ---- device-resident Krylov loops (fb_graph.cu) ---------------------------
 * A CUDA graph holding one conditional WHILE node; the body is captured from
 * a stream (begin / launches of one solver iteration / end) and the loop is
 * continued or stopped on the device by the check kernel. */
typedef struct fb_while_graph fb_while_graph;
int fb_while_graph_create(fb_while_graph** out);
unsigned long long fb_while_graph_handle(const fb_while_graph* G);
int fb_while_graph_begin(fb_while_graph* G, void* stream);
int fb_while_graph_end(fb_while_graph* G, void* stream);
int fb_while_graph_launch(const fb_while_graph* G, void* stream);
void fb_while_graph_destroy(fb_while_graph* G);
/* PCG stopping test of solvers.py:141-165 on device scalars s = [rz, pAp,
 * alpha, rz_new, beta]: state = [iterations, stop reason, max_iters],
 * hist[it] = relres, cfg = [norm0, rel_tol]; in a graph (in_graph = 1) it
 * sets the WHILE condition, pausing before every `period`-th iteration. */
int fb_cg_check(unsigned long long handle, int in_graph, double* s_dev, int* state_dev,
                double* hist_dev, const double* cfg_dev, int period, void* stream);
/* p = z + beta_dev[0] p */
int fb_xpby_dev(int64_t n, const double* z_dev, const double* beta_dev, double* p_dev,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FBB200_H */
