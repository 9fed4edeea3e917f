/* trihalo_b200 — C ABI of the B200-native halo interpolation / restriction path.
 *
 * This is the drop-in boundary for the reference's per-face operator API
 * (/root/reference/pkg/src/trihalo/schemes.py).  The reference is pure Python
 * and has no FFI of its own; these entry points are what a host code (the
 * Python mirror in paper_2504_15814_b200/, or a C++ AMR driver) binds to
 * replace, one for one:
 *
 *   th_operator_create       OperatorCache.get / build_reference_operator
 *                            (taylor.py:252-308, schemes.py:56-70), plus the
 *                            tensor-product axis matrices of HaloExchange.__init__
 *                            (schemes.py:155-169).  One operator per
 *                            (role, scheme, p, k); segment / half are chosen per
 *                            face at apply time instead of per operator.
 *   th_apply_faces           HaloExchange.run (schemes.py:185-202), batched over
 *                            many faces; interpolate_halo / restrict_halo /
 *                            apply_scheme (schemes.py:73-116) are one-face calls.
 *   th_csr_apply             csr.apply / csr._apply_kernel (csr.py:143-173) on
 *                            reference-frame buffers.
 *   th_operator_export_rows  CsrOperator rows of a segment / half row block
 *                            (csr.py:176-248), for parity checks and dumps.
 *   th_scheme_feasible       scheme_feasible (schemes.py:23-47).
 *   th_copy_faces            same-level halo fill between patches of one level
 *                            (outside the reference).
 *   th_copy_boxes            strided cell-box copies: packing / unpacking the
 *                            source boxes of faces whose coarse and fine patches
 *                            live on different GPUs (outside the
 *                            reference, which is single-process).
 *   th_operator_source_box   the source cells an operator's kernels read for
 *                            one segment / half (the box a cross face ships).
 *   th_pseudoinverse_rows    solve_pseudoinverse_rows (linalg.py:99-112), the
 *                            builder's least-squares fit (build_derivative_fit).
 *
 * Conventions
 *   - Cell data are AoS: the u unknowns of a cell are contiguous (stride 1),
 *     exactly the reference HaloBuffer layout (geometry.py:272-303).  Cells
 *     are addressed through per-face element offsets and per-axis element
 *     strides, so the same call serves the reference's contiguous world
 *     halo buffers and a patch pool with halos.
 *   - All device pointers are plain CUDA device pointers; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).  Calls
 *     are asynchronous on that stream.
 *   - Return codes map onto the reference exception classes (errors.py):
 *     TH_OK, TH_ERR_CONFIG (ConfigurationError), TH_ERR_INFEASIBLE
 *     (StencilInfeasibleError), TH_ERR_CONTRACT (ContractViolationError),
 *     TH_ERR_SINGULAR (SingularFitError), TH_ERR_CUDA (device failure).
 *     th_last_error() returns the message of the last failing call on the
 *     calling thread; th_last_error_column() the SingularFitError column.
 */
#ifndef TRIHALO_B200_H
#define TRIHALO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TH_OK = 0,
  TH_ERR_CONFIG = 1,
  TH_ERR_INFEASIBLE = 2,
  TH_ERR_CONTRACT = 3,
  TH_ERR_SINGULAR = 4,
  TH_ERR_CUDA = 5
};

enum { TH_ROLE_INTERPOLATE = 0, TH_ROLE_RESTRICT = 1 };

enum {
  TH_SCHEME_TENSOR_LINEAR = 0, /* schemes.py:19 "tensor_linear" */
  TH_SCHEME_MATRIX_LINEAR = 1, /* "matrix_linear" */
  TH_SCHEME_ORDER2 = 2,        /* "order2" */
  TH_SCHEME_ORDER3 = 3         /* "order3" */
};

enum { TH_HALF_FULL = 0, TH_HALF_INNER = 1, TH_HALF_OUTER = 2 };

/* One face of a batch.  Offsets and strides are in elements (doubles).
 * World axes are x=0, y=1, z=2 (geometry.py:39).
 *
 * Interpolation (role 0): the source is the world region
 *   interp_source_shape(cfg) (geometry.py:244-246): 2k coarse cells along
 *   the normal by p x p tangentially; src[0] is the offset of its world
 *   low-corner cell, src[1..8] are unused.  The target is segment `segment`'s
 *   k x p x p fine block, interp_target_shape(cfg) (geometry.py:249-256);
 *   dst is the offset of its world low-corner cell.
 * Restriction (role 1): the source is restrict_source_shape(cfg)
 *   (geometry.py:259-261), 2k x 3p x 3p fine cells, split tangentially into
 *   the 3 x 3 blocks of the nine fine patches; src[b1 + 3*b2] is the offset of
 *   the world cell (normal 0, t1 = b1*p, t2 = b2*p) — i.e. the low corner of
 *   fine block (b1, b2) — with t1 < t2 the two tangential world axes.  For a
 *   contiguous source buffer src[s] = base + b1*p*stride[t1] + b2*p*stride[t2].
 *   The target is restrict_target_shape(cfg, half) (geometry.py:264-265).
 * The unknown index is stride 1 in both source and target storage.
 */
typedef struct th_face {
  int64_t src[9];
  int64_t dst;
  int64_t src_stride[3];
  int64_t dst_stride[3];
  int32_t normal;  /* 0, 1, 2 */
  int32_t side;    /* 0 = coarse on the negative side, 1 = positive */
  int32_t segment; /* interpolation only: 0..8 */
  int32_t half;    /* restriction only: TH_HALF_* */
} th_face;

/* One cell box for th_copy_boxes: ext[0] x ext[1] x ext[2] cells (world x, y, z)
 * at element offset src (strides src_stride, per world axis) copied to element
 * offset dst (strides dst_stride); u unknowns per cell, unknown stride 1. */
typedef struct th_box {
  int64_t src;
  int64_t dst;
  int64_t src_stride[3];
  int64_t dst_stride[3];
  int32_t ext[3];
  int32_t pad;
} th_box;

typedef struct th_operator th_operator;

typedef struct th_operator_info {
  int32_t role, scheme, p, k;
  int32_t n_src_cells;       /* reference source region cells */
  int32_t n_tgt_cells_full;  /* full-face / full-target rows */
  int32_t n_blocks;          /* distinct dense weight blocks uploaded */
  int32_t max_items_per_face;
  int64_t device_bytes;      /* uploaded operator bytes */
  double max_condition;      /* Taylor fits: max |R_ii| ratio (taylor.py:160-168) */
  int32_t n_condition_warnings;
  int32_t kernel;            /* kernel family chosen for this operator */
} th_operator_info;

/* library / device */
int32_t th_abi_version(void);
const char* th_last_error(void);
int32_t th_last_error_column(void);

/* feasibility (schemes.py:23-47): returns TH_OK when feasible, TH_ERR_INFEASIBLE
 * with th_last_error() naming the constraint, TH_ERR_CONFIG on bad arguments */
int32_t th_scheme_feasible(int32_t role, int32_t scheme, int32_t p, int32_t k);

/* host construction + upload to the current CUDA device */
int32_t th_operator_create(int32_t role, int32_t scheme, int32_t p, int32_t k, th_operator** out);
/* host construction only (no device upload): info and row export work, apply
 * returns TH_ERR_CONTRACT.  Lets a CPU-only process inspect the operators. */
int32_t th_operator_create_host(int32_t role, int32_t scheme, int32_t p, int32_t k, th_operator** out);
void th_operator_destroy(th_operator* op);
int32_t th_operator_info_get(const th_operator* op, th_operator_info* info);

/* Export the operator's rows for a segment (interpolation, 0..8, or -1 for
 * the full face) or half (restriction, TH_HALF_*), in the reference's row
 * order and reference-source column numbering, entries with |w| >= 1e-14
 * (csr.py:20).  Two-phase: call with NULL arrays to get nnz/rows, then again
 * with row_offsets[n_rows+1], col_indices[nnz], values[nnz].  Host memory.
 * tensor_linear operators export the collapsed product of their axis rows. */
int32_t th_operator_export_rows(const th_operator* op, int32_t selector, int64_t* n_rows, int64_t* nnz,
                                int64_t* row_offsets, int64_t* col_indices, double* values);

/* Apply the operator to n_faces faces.  faces points to DEVICE memory
 * (n_faces th_face records).  `flag`, if not NULL, is a device int32 that is
 * OR-ed with 1 when a non-finite source value feeds the faces (the reference raises
 * ContractViolationError for non-finite sources, schemes.py:186).  The interpolation kernels
 * check each source slice through its first Gram moment (a plain sum), so finite inputs whose
 * sum overflows (|v| ~ 1e307) are flagged too; the restriction kernels check every produced
 * value.  th_check_finite checks values one by one. */
int32_t th_apply_faces(const th_operator* op, const double* src, double* dst, const th_face* faces,
                       int64_t n_faces, int32_t u, int32_t* flag, void* stream);

/* Check that every value of a device buffer is finite: OR-s 1 into *flag
 * otherwise (the whole-source check of schemes.py:186 / csr.py:165). */
int32_t th_check_finite(const double* values, int64_t n, int32_t* flag, void* stream);

/* Normal source layers an operator reads, in reference order [lo, lo + count)
 * of the 2k source layers (the union of its stencil windows).  World layers are
 * the same for coarse side 0 and mirrored (2k - lo - count) for side 1. */
int32_t th_operator_support_layers(const th_operator* op, int32_t* lo, int32_t* count);

/* Asynchronous copy of n_faces back-to-back world boxes (x fastest, u unknowns
 * per cell, extent n_ext along `normal`, t_ext along the two tangential axes)
 * restricted to the normal layers [lo, lo + count): one cudaMemcpy2DAsync /
 * cudaMemcpy3DAsync for the whole group.  kind: 0 host->device, 1 device->host
 * (host memory should be pinned).  Used to ship only an operator's support
 * from host buffers in the reference layout. */
int32_t th_copy_box_layers(const double* src, double* dst, int64_t n_faces, int32_t normal, int32_t n_ext,
                           int32_t t_ext, int32_t u, int32_t lo, int32_t count, int32_t kind, void* stream);

/* Same-level halo copy (no reference counterpart: the reference
 * handles 3:1 faces only, so this is the part of a time step's halo fill between two
 * patches of the same level).  Face f copies the n_ext x t_ext x t_ext world box of
 * cells (n_ext along faces[f].normal) at src + faces[f].src[0] (world strides
 * faces[f].src_stride) to dst + faces[f].dst (strides faces[f].dst_stride), u unknowns
 * per cell, unknown stride 1.  Bit-exact copy.  src and dst may be the same pool when no
 * face's target box overlaps ANY face's source box of the same launch (the kernel reads
 * through the non-coherent path while other faces write): pool_same_level_faces with
 * 1 <= k <= p satisfies it (halo layers are written, interior layers read).  All pointers
 * device. */
int32_t th_copy_faces(const double* src, double* dst, const th_face* faces, int64_t n_faces, int32_t n_ext,
                      int32_t t_ext, int32_t u, void* stream);

/* Least-squares pseudo-inverse rows of a full-rank tall s x n matrix (host, row-major):
 * w (n x s, row-major) = R^-1 Q^T from a Householder QR without pivoting, *cond = max|R_ii| /
 * min|R_ii|; TH_ERR_SINGULAR (th_last_error_column() = column) when a pivot is below 1e-12 of
 * the largest, TH_ERR_CONTRACT for s < n or non-finite entries.  The builder's own fit
 * (linalg.py:40-112 solve_pseudoinverse_rows), exported for build_derivative_fit. */
int32_t th_pseudoinverse_rows(const double* a, int32_t s, int32_t n, double* w, double* cond);

/* Asynchronous byte copy on `stream`: kind 0 host->device, 1 device->host, 2 device->device
 * (host memory pinned or registered).  Moves patch pools and results between host buffers and
 * HBM for callers that hold their data on the host. */
int32_t th_memcpy_async(void* dst, const void* src, int64_t bytes, int32_t kind, void* stream);

/* Copy the same set of blocks out of n_patches consecutive patches (host <-> device, kind as
 * th_memcpy_async): a patch is patch_elems doubles, seen as rows of row_elems doubles; block b
 * = blocks[4b .. 4b+3] = {first row, rows, first element in the row, elements per row}.  One
 * cudaMemcpy3DAsync per block (rows x patches).  Ships only the cells a sweep reads from a
 * patch pool held in host memory. */
int32_t th_copy_patch_blocks(void* dst, const void* src, int64_t n_patches, int64_t patch_elems, int64_t row_elems,
                             const int32_t* blocks, int32_t n_blocks, int32_t kind, void* stream);

/* Pack (pack = 1: pool -> compact) or unpack (0: compact -> pool) the same blocks of n_patches
 * consecutive patches, all device memory.  blocks (device, int32 [n_blocks][4], the format of
 * th_copy_patch_blocks); block_offsets (device, int64 [n_blocks]) = each block's element offset
 * inside a patch's compact record of compact_elems elements.  Lets a host hold only the cells a
 * sweep reads, contiguously, and ship them with plain copies. */
int32_t th_pool_blocks(double* pool, double* compact, int64_t n_patches, int64_t patch_elems, int64_t row_elems,
                       const int32_t* blocks, const int64_t* block_offsets, int32_t n_blocks, int64_t compact_elems,
                       int32_t pack, void* stream);

/* Copy n_boxes cell boxes (th_box records in DEVICE memory) from src to dst, both
 * device.  Targets may overlap one another only where they write identical values
 * (the multi-GPU unpack writes one fine patch's boxes for several orientations into
 * one staging slot); no target may overlap a source of the same launch.  Bit-exact. */
int32_t th_copy_boxes(const double* src, double* dst, const th_box* boxes, int64_t n_boxes, int32_t u,
                      void* stream);

/* Union of the source windows the kernels read for one face selection, in
 * reference source coordinates: box = {lo0, count0, lo1, count1, lo2, count2}
 * along (normal, t1, t2) of the reference source region (interpolation: 2k x p x p,
 * selector = segment 0..8; restriction: 2k x 3p x 3p, selector = TH_HALF_*).
 * Every source cell outside the box is never read, so a face whose source
 * arrives from another GPU needs only this box. */
int32_t th_operator_source_box(const th_operator* op, int32_t selector, int32_t* box);

/* CSR apply on reference-frame AoS buffers (csr.py:143-173); all pointers device. */
int32_t th_csr_apply(const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                     int64_t n_rows, const double* src, double* out, int32_t u, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TRIHALO_B200_H */
