/*
 * zt.h — C ABI of the B200-native isospectral time-step hot path
 * (Zeitlin–Euler on the sphere, arXiv 2206.05466).
 *
 * One shared library (paper_2206_05466_b200/libzt.so, sm_100a).  Every entry
 * point takes plain device pointers and sizes, enqueues on the caller's
 * cudaStream_t (passed as void*), never allocates inside a step call (the
 * workspace is caller-owned), and returns a zt_status code; details of the
 * last failure on the calling thread are in zt_last_error().
 *
 * Matrices are complex128, row-major, interleaved (re, im) doubles, with a
 * leading dimension counted in complex elements — i.e. numpy/torch
 * complex128 C-order memory, zero-copy.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/zeitlin/):
 *   zt_op_create        laplacian.py:179-219, 319-322  LaplacianOperator / build_operator
 *   zt_stream_solve     laplacian.py:370-431 (+272-316) solve_stream (check=False body)
 *   zt_apply_laplacian  laplacian.py:341-367            apply_laplacian
 *   zt_residuals        laplacian.py:75-104             skewness_residual / trace_residual
 *   zt_fixed_point      integrator.py:96-138            fixed_point_solve
 *   zt_midpoint_step    integrator.py:141-171           midpoint_step_info
 *   zt_zgemm            integrator.py:127-128, 155-156  the numpy `@` products (OpenBLAS zgemm)
 *   zt_commutator /     integrator.py:127-129           (a - a^H) and the sandwich update
 *   zt_sandwich
 *   zt_basis_vectors    basis.py:119-165 compute_basis    the quantized basis eigenvectors
 *   zt_basis_extract    basis.py:319-331 extract          per-diagonal transforms
 *   zt_basis_project    basis.py:276-316 project
 *   zt_grid_eval        diagnostics.py:113-187 evaluate_on_grid
 */
#ifndef ZT_H_
#define ZT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ZT_OK = 0,
  ZT_EINVAL = 1,      /* bad argument (maps to ValueError) */
  ZT_ESTRUCTURE = 2,  /* input not skew-Hermitian / traceless (StructureError) */
  ZT_ENOCONV = 3,     /* fixed point did not reach tol (FixedPointError) */
  ZT_ELINALG = 4,     /* tridiagonal factorisation failed (LinAlgError) */
  ZT_ECUDA = 5,       /* CUDA runtime error */
  ZT_ENCCL = 6,       /* collective failure */
  ZT_ENOMEM = 7       /* workspace too small / allocation failed */
} zt_status;

typedef struct zt_operator* zt_op_t;

int zt_version(void);
const char* zt_strerror(int status);
const char* zt_last_error(void);

/* Per-N Laplacian operator on `device` (laplacian.py:179-219).  Builds the
 * per-chunk LDL^T carry tables on the GPU; immutable afterwards and
 * shareable across streams.  n >= 2. */
int zt_op_create(int n, int device, zt_op_t* op);
int zt_op_destroy(zt_op_t op);
int zt_op_n(zt_op_t op);
/* Copies the reference-layout factor tables (sheared N x N, laplacian.py:
 * 213-215) to host arrays (test hook; either pointer may be NULL). */
int zt_op_factors(zt_op_t op, double* linv_host, double* dinv_host);

/* P = lap^{-1} W for `batch` matrices (laplacian.py:370-431, check=False).
 * Reads only the lower triangle + diagonal of W; writes the full P (lower
 * from the solve, strict upper by skew reflection, laplacian.py:306-316).
 * W and P must not alias.  Strides between batch entries in complex elems. */
int zt_stream_solve(zt_op_t op, const double* w, int64_t ldw, int64_t stride_w, double* p,
                    int64_t ldp, int64_t stride_p, int batch, void* stream);

/* Same with caller-owned carry workspace of zt_solve_workspace_bytes(n,
 * batch) bytes (no allocation; graph-capturable). */
size_t zt_solve_workspace_bytes(int n, int batch);
int zt_stream_solve_ws(zt_op_t op, const double* w, int64_t ldw, int64_t stride_w, double* p,
                       int64_t ldp, int64_t stride_p, int batch, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Y = sign * stencil(W) over diagonals (laplacian.py:341-367), sign = +-1;
 * lower triangle of W read only; bit-identical to the reference. */
int zt_apply_laplacian(zt_op_t op, const double* w, int64_t ldw, int64_t stride_w, double* y,
                       int64_t ldy, int64_t stride_y, int sign, int batch, void* stream);

/* out_dev[0] = ||W + W^H||_F / ||W||_F, out_dev[1] = |tr W| / ||W||_F,
 * out_dev[2] = ||W||_F (device doubles; 0,0,0 for the zero matrix). */
int zt_residuals(int n, const double* w, int64_t ldw, double* out_dev, void* stream);
size_t zt_resid_workspace_bytes(int n);
int zt_residuals_ws(int n, const double* w, int64_t ldw, double* out_dev, void* workspace,
                    void* stream);

/* C = A @ B (complex128, n x n, all row-major).  `algo` 0 = 3M (Gauss)
 * DMMA, 1 = 4M DMMA.  Used by the GEMM op benchmark and casimirs. */
int zt_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
             int64_t ldc, int algo, void* stream);

/* Rectangular C (m x n) = A (m x k) @ B (k x n), row-major, 16B-aligned
 * operands (the local products of the sharded step). */
int zt_zgemm_rect(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb,
                  double* c, int64_t ldc, int algo, void* stream);

/* Row-block update of the sharded step (rows R of the N x N update held
 * by one rank): b = a_R @ P (a_R: m x n, P: n x n); out = base +
 * hh (a_R - ah_R) + qq b where ah_R = rows R of a^H; *resid_dev (device
 * uint64, zeroed by the caller) receives the bit pattern of
 * max|out - xprev| (NaN-propagating).  All row blocks use leading dim ld. */
int zt_zgemm_update_rows(int m, int n, const double* a_rows, const double* p,
                         const double* ah_rows, const double* base, const double* xprev,
                         double* out, int64_t ld, double hh, double qq,
                         unsigned long long* resid_dev, void* stream);

/* Workspace for zt_fixed_point / zt_midpoint_step at size n (bytes). */
size_t zt_step_workspace_bytes(int n);

/* Fixed-point solve for W~ (integrator.py:96-138).  wt receives W~;
 * *iterations / *residual report the loop; returns ZT_ENOCONV (with both
 * filled) when max_iter is exhausted, ZT_ESTRUCTURE when W_n fails the
 * 1e-10 skew/trace gate (laplacian.py:107-116).  Synchronises the stream
 * once per iteration (4-byte residual read-back). */
int zt_fixed_point(zt_op_t op, const double* wn, double* wt, double h, double tol, int max_iter,
                   void* workspace, size_t workspace_bytes, int* iterations, double* residual,
                   void* stream);

/* One midpoint step (integrator.py:141-171): w_next = W_{n+1} from w_n with
 * h_eff = h * comm_scale.  If consistency != NULL it receives
 * max|W~ - (h/2)(a-a^H) - (h^2/4) a P~ - W_n| (integrator.py:160-163).
 * w_next must not alias w_n. */
int zt_midpoint_step(zt_op_t op, const double* wn, double* w_next, double h_eff, double tol,
                     int max_iter, void* workspace, size_t workspace_bytes, int* iterations,
                     double* residual, double* consistency, void* stream);

/* zt_midpoint_step that also delivers W_{n+1} to host memory `host_out`
 * (n*n complex128, page-locked for overlap), as the reference's
 * midpoint_step_info returns a fresh numpy array (integrator.py:165-171).
 * With the step graph, the final update's GEMM writes W_{n+1} tile pair by
 * tile pair and publishes each 64-row block; a copy stream waits on those
 * flags (cuStreamWaitValue32) and moves the blocks while the GEMM runs.
 * Returns after the copy completed; w_next holds W_{n+1} as well. */
int zt_midpoint_step_host(zt_op_t op, const double* wn, double* w_next, double* host_out, double h_eff,
                          double tol, int max_iter, void* workspace, size_t workspace_bytes,
                          int* iterations, double* residual, void* stream);

/* INT8 tensor-core building block of an FP64-accurate complex GEMM
 * (Ozaki scheme II with a Gaussian-integer split, csrc/zt_oz.cu).  Every
 * modulus p_j (odd, prime factors = 1 mod 4, zt_oz_moduli) has a square root
 * iota_j of -1 (zt_oz_iotas), so a complex residue product is two real ones:
 * given centred int8 planes A [nmod][2][mp][kp] = (phi+, phi-) and
 * B [nmod][2][np][kp] (K-major rows of B^T), with U = A+ B+^T and
 * V = A- B-^T (exact int32 accumulation in TMEM, tcgen05 kind::i8 MMAs on
 * CTA pairs), R [nmod][2][mp][np] receives ((U + V) + k_j) mod p_j and
 * ((U - V) + k_j) mod p_j, k_j = (p_j - 1) / 2, unsigned bytes in [0, p_j).
 * For phi+- = re +- iota_j im (mod p_j) of complex matrices A, B this is
 * 2 Re(A B^T) and 2 iota_j Im(A B^T) mod p_j.  mp, np multiples of 256, kp
 * of 128; lower != 0: square, only the 256-tiles on or below the diagonal.
 * zt_oz_moduli / zt_oz_iotas write the moduli / roots, return their count. */
int zt_oz_modgemm(int nmod, int mp, int np, int kp, const void* a, const void* b, void* r, int lower,
                  void* stream);
int zt_oz_moduli(int* out, int cap);
int zt_oz_iotas(int* out, int cap);
/* C = A B (complex128, n x n, row-major with leading dimensions) through the
 * residue GEMM: rows of A and columns of B scaled to integers of
 * zt_oz_bits(n) bits (55 up to n = 4096, 54 above), 17 moduli <= 241, exact
 * CRT reconstruction in FP64 pieces; a
 * row of A or column of B holding a NaN or an infinity gives a NaN row /
 * column of C.  bmode 1: B is
 * skew-Hermitian with B[k][j] == -conj(B[j][k]) exactly off the diagonal
 * (converted row-wise, no transpose).  lower: only the 256-tiles of C on or
 * below the diagonal.  workspace: zt_oz_workspace_bytes(n). */
size_t zt_oz_workspace_bytes(int n);
/* CUDA-event totals of the residue-GEMM launches recorded while profiling
 * (zt_profile_enable): ms/counts [0] full products, [1] lower-triangle ones. */
int zt_oz_profile_read(double* ms, long long* counts, int reset);
int zt_oz_zgemm(int n, const double* a, int64_t lda, const double* b, int64_t ldb, int bmode, double* c,
                int64_t ldc, int lower, void* workspace, size_t workspace_bytes, void* stream);

/* Building blocks of the row-block sharded step on the INT8 product
 * (paper_2206_05466_b200/sharded.py): no reference
 * counterpart (the reference is single-process; the paper's
 * distributed products are ScaLAPACK pzgemm).
 *   zt_oz_bits(K): integer bits per operand entry for inner dimension K.
 *   zt_oz_plane_bytes(rows, cols): bytes of one residue-plane set
 *     [17][2][pad(rows)][pad(cols)], pad = multiple of 256.
 *   zt_oz_convert_rows: rows x kdim block (row-major, ld) to planes; mode 0
 *     A operand, mode 1 skew-B operand of a skew-Hermitian matrix whose
 *     diagonal entry of local row j is column diag0 + j, mode 2 both (A
 *     planes into planes, skew-B into planes2) from one read; shift:
 *     pad(rows) ints.
 *   zt_oz_convert_cols: kdim x ncols matrix as a general B operand
 *     (column scales); colmax_ws: pad(ncols) 8-byte words.
 *   zt_oz_reconstruct: residues of zt_oz_modgemm(…, pad(m), pad(n), …) to
 *     complex128 C (m x n) into c (nullable), and/or column j into
 *     ((double*)peers[j / mloc]) at row r0 + i of an N x mloc block (the
 *     all-to-all fused into the reconstruction), and/or -conj(C)^T into
 *     mirror (ld_mirror); lower != 0 (square, residues of a lower-mode
 *     zt_oz_modgemm): only the 256-tiles on or below the diagonal, entries of
 *     strictly-lower tiles mirrored (pass the block itself as mirror to
 *     complete a skew-Hermitian diagonal block). */
int zt_oz_bits(int k);
size_t zt_oz_plane_bytes(int rows, int cols);
int zt_oz_convert_rows(int rows, int kdim, const double* src, int64_t ld, int mode, int diag0, int kb, void* planes,
                       int* shift, void* planes2, void* stream);
int zt_oz_convert_cols(int kdim, int ncols, const double* src, int64_t ld, int kb, void* planes, int* shift,
                       void* colmax_ws, void* stream);
int zt_oz_reconstruct(int m, int n, const void* r, const int* rs, const int* cs, double* c, int64_t ldc,
                      const unsigned long long* peers, int mloc, int r0, double* mirror, int64_t ld_mirror,
                      int lower, void* stream);

/* Config-3 ops (integrator.py:127-129): commutator C = P W - W P = a - a^H
 * with a = P W; sandwich S = W - (h/2)(a - a^H) - (h^2/4) a P
 * = (I - hP/2) W (I + hP/2).  `work` holds n*n complex (a). */
int zt_commutator(int n, const double* p, const double* w, double* c, double* work, void* stream);
int zt_sandwich(int n, const double* p, const double* w, double h, double* s, double* work,
                void* stream);

/* Peer-memory variants of the sharded step (rank r0 / mloc = N / G): the
 * collectives are stores in the GEMM epilogues to NVLink peer-mapped buffers
 * (`peers`: device array of npeer pointers, one per rank, e.g. from
 * torch symmetric memory), visible to the peers after the kernel completes
 * and a rank barrier.
 *   zt_zgemm_rect_scatter      a_R = P_R X; column block h of a_R also to
 *                              rank h's N x mloc buffer a[:, R_h] (all-to-all)
 *   zt_zgemm_update_rows_peer  the row-block update with (a^H)_R read from
 *                              this rank's a[:, R] buffer; the new rows also
 *                              to every rank's N x N iterate (all-gather)
 *   zt_rows_broadcast          a row block into every rank's N x N buffer
 *   zt_zgemm_rect_mirror       C = A B and -conj(C^T) into `mirror` (the
 *                              partner rank's rows of the skew-Hermitian
 *                              b = a P, so each block pair is computed once);
 *                              mirror == NULL and m == n: a diagonal block,
 *                              lower tiles only, mirrored in place
 *   zt_update_rows_ew          the row-block update from a precomputed b_R,
 *                              residual, new rows broadcast to every rank */
int zt_zgemm_rect_scatter(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb,
                          double* c, int64_t ldc, const unsigned long long* peers, int npeer, int r0, int mloc,
                          void* stream);
int zt_zgemm_update_rows_peer(int m, int n, const double* a_rows, const double* p, const double* acol, int mloc,
                              const double* base, const double* xprev, double* out, int64_t ld, double hh,
                              double qq, unsigned long long* resid, const unsigned long long* peers, int npeer,
                              int r0, void* stream);
int zt_rows_broadcast(int m, int n, const double* rows, int64_t ld, const unsigned long long* peers, int npeer,
                      int r0, void* stream);
int zt_zgemm_rect_mirror(int m, int n, int k, const double* a, int64_t lda, const double* b, int64_t ldb,
                         double* c, int64_t ldc, double* mirror, int64_t ld_mirror, void* stream);
int zt_update_rows_ew(int m, int n, const double* a_rows, const double* acol, int mloc, const double* b_rows,
                      const double* base, const double* xprev, double* out, int64_t ld, double hh, double qq,
                      unsigned long long* resid, const unsigned long long* peers, int npeer, int r0, void* stream);

/* Device-driven fixed point for callers that enqueue their own update (the
 * sharded step, sharded.py): a CUDA graph captured from `stream` whose
 * fixed-point loop is a conditional WHILE node (the single-GPU step's
 * scheme, integrator.py:125-138), so a step is one graph launch with no host
 * round trip per update.
 *   zt_loop_graph_begin      begin capturing `stream` (the prologue); the
 *                            loop condition starts at 1
 *   zt_loop_graph_gate       the input gate (laplacian.py:107-116) on the
 *                            two residuals at val[0..1] (zt_residuals
 *                            output): a rejected W_n runs no update
 *   zt_loop_graph_body_begin append the WHILE node and capture `body` into
 *                            its body graph (the update goes here)
 *   zt_loop_graph_decide     in the body: r = max of `nslots` residual bit
 *                            patterns (one per rank, NaN above every
 *                            number), mail[2] += 1, mail[3] = r; continue
 *                            while !(r <= tol) and mail[2] < max_iter
 *   zt_loop_graph_body_end   end the body capture
 *   zt_loop_graph_end        end the capture and instantiate
 *   zt_loop_graph_launch / zt_loop_graph_destroy
 *   zt_peer_put_u64          *src into dst_ptrs[h][index] for every rank h
 *                            (dst_ptrs: device array of peer pointers),
 *                            then a system-scope fence */
typedef struct zt_loop_graph* zt_loop_graph_t;
int zt_loop_graph_begin(void* stream, zt_loop_graph_t* out);
int zt_loop_graph_gate(zt_loop_graph_t g, const double* val, void* stream);
int zt_loop_graph_body_begin(zt_loop_graph_t g, void* stream, void* body);
int zt_loop_graph_decide(zt_loop_graph_t g, const unsigned long long* slots, int nslots, unsigned long long* mail,
                         double tol, int max_iter, void* body);
int zt_loop_graph_body_end(zt_loop_graph_t g, void* body);
int zt_loop_graph_end(zt_loop_graph_t g, void* stream);
int zt_loop_graph_launch(zt_loop_graph_t g, void* stream);
int zt_loop_graph_destroy(zt_loop_graph_t g);
int zt_peer_put_u64(const unsigned long long* src, const unsigned long long* dst_ptrs, int index, int npeer,
                    void* stream);

/* Quantized spherical-harmonic basis (basis.py).
 * Vectors for orders m0 <= m < m1 are stored like the reference's
 * QuantizedBasis.vectors[m]: row-major (N - m) x n_l(m) doubles,
 * n_l(m) = N - max(m, 1), columns l = max(m,1)..N-1, at vec + off[m]
 * (device int64 offsets, indexed by absolute m).  Coefficients are complex
 * (interleaved), order m at pos/neg + 2 * coff[m] (n_l(m) entries each).
 *   zt_basis_vectors   compute_basis eigenvectors, sign rule of
 *                      basis.py:110-114 (basis.py:119-165)
 *   zt_basis_extract   w_lm = -i Tr(T_lm^H W) for both signs of m
 *                      (basis.py:319-331)
 *   zt_basis_project   W = sum i w_lm T_lm into the rows/columns of the
 *                      m-diagonals; neg == NULL: skew completion of the
 *                      lower triangle (basis.py:276-316) */
int zt_basis_vectors(int n, int m0, int m1, const long long* off, double* vec, void* stream);
int zt_basis_extract(int n, int m0, int m1, const long long* off, const long long* coff,
                     const double* vec, const double* w, int64_t ldw, double* pos, double* neg,
                     void* stream);
int zt_basis_project(int n, int m0, int m1, const long long* off, const long long* coff,
                     const double* vec, const double* pos, const double* neg, double* w,
                     int64_t ldw, void* stream);

/* Grid rendering (diagnostics.py:113-187): the real
 * field sum_lm w_lm Y_lm on theta_i = i pi / (nlat-1), phi_j = 2 pi j / nlon
 * is the real part of the complex nlat x nlon `field`; `work` holds
 * (nlat + nlon) x (lmax + 1) complex. */
int zt_grid_eval(int n, int lmax, int nlat, int nlon, const long long* coff, const double* pos,
                 double* work, double* field, void* stream);

/* Per-kernel device timing for the roofline report: when enabled, CUDA
 * events bracket the stream solve, GEMM-1 (a = P X) and GEMM-2 (update) of
 * every update inside zt_midpoint_step; zt_profile_read returns the summed
 * milliseconds and launch counts [solve, gemm1, gemm2]. */
int zt_profile_enable(int on);
int zt_profile_read(double* ms3, int64_t* counts3, int reset);

/* Number of kernels this library launched since load (device-side work
 * evidence for the bench's gpu_launches claim). */
int64_t zt_launch_count(void);

/* Step execution mode for zt_midpoint_step / zt_midpoint_step_host: 1 (the
 * default, or ZT_GRAPH unset/1) runs each step as one CUDA graph with the
 * fixed point as a conditional WHILE node; 0 launches the same kernels
 * eagerly with one 8-byte read-back per iteration (results are bitwise
 * identical).  Returns the previous mode. */
int zt_set_graph(int on);

/* The step's product path, fixed when the library loads: 2 = the INT8
 * Ozaki-II product (default), 0 / 1 = native FP64 DMMA 3M / 4M
 * (ZT_GEMM_ALGO=3m / 4m). */
int zt_step_algo(void);

#ifdef __cplusplus
}
#endif
#endif /* ZT_H_ */
