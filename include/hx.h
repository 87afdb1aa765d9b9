/* hx.h — C ABI of the B200 H x H product library (libhx.so).
 *
 * Drop-in boundary for the reference's product path.  The reference seam is the Python
 * call ``hmult_new(h, k, cfg)`` (/root/reference/pkg/src/hmat/multiply.py:252-256), whose
 * recursion ``_multiply``/``rec`` (multiply.py:207-249) drives ``restrict``
 * (sumexpr.py:136-154), ``_thin_product`` (sumexpr.py:93-117), ``evaluate_dense``
 * (sumexpr.py:165-170) and one ``compress`` per far leaf (compressors.py:441-452).
 * A per-block crossing at the ``compress`` seam would mean 1e5..1e6 Python->C calls, so
 * this library replaces the whole product: the host wrapper
 * (paper_1805_08998_b200/multiply.py) keeps the reference signature and calls, in order,
 *
 *   hx_plan_create      restrict/_thin_product bookkeeping     -> flat term lists
 *   hx_ctx_create       device context (one per GPU / process)
 *   hx_ctx_operand      upload (or attach) the packed A / B pools   (HMatrix.data)
 *   hx_product          term formation, materialization, recompression (_multiply)
 *   hx_result_*         ranks, degraded flags and factors back to the caller
 *
 * plus the GPU operand assembly that replaces assemble_hmatrix (hmatrix.py:97-118).
 * All entry points return 0 on success or a negative hx_status; hx_last_error() gives
 * the message.  Plain C types only; no torch types cross this boundary.
 */
#ifndef HX_H
#define HX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum hx_status {
  HX_OK = 0,
  HX_EINVAL = -1,      /* bad argument / config  -> ValueError   */
  HX_ENOMEM = -2,      /* device or host allocation failed -> MemoryError */
  HX_ECUDA = -3,       /* CUDA runtime error     -> RuntimeError */
  HX_EUNSUPPORTED = -4 /* valid input this build does not handle -> NotImplementedError */
};

/* Block-cluster tree in array form (clustering.py:110-172): cluster ids and block ids in
 * the reference's DFS pre-order; children ordered tau-child-major like the reference. */
typedef struct hx_tree {
  int32_t n_clusters;
  const int64_t* c_lo;     /* [n_clusters] first tree position                      */
  const int64_t* c_hi;     /* [n_clusters] one past the last position               */
  const int32_t* c_child;  /* [2 * n_clusters] children, -1 for a leaf cluster       */
  int32_t n_nodes;
  const int32_t* tau;      /* [n_nodes] row cluster id                              */
  const int32_t* sigma;    /* [n_nodes] column cluster id                           */
  const int8_t* kind;      /* [n_nodes] 0 inner, 1 far, 2 near                      */
  const int32_t* child;    /* [4 * n_nodes] children, -1 when the node is a leaf    */
} hx_tree;

/* Leaf payload directory of one H-matrix operand (HMatrix.data, hmatrix.py:48-65) over a
 * packed float64 pool: low-rank leaves store left (m x k) then right (n x k), dense
 * leaves store m x n, all column-major. */
typedef struct hx_operand {
  const int8_t* payload;   /* [n_nodes] 0 none (inner), 1 low rank, 2 dense          */
  const int32_t* rank;     /* [n_nodes] rank of low-rank leaves                      */
  const int64_t* u_off;    /* [n_nodes] element offset of left factor                */
  const int64_t* v_off;    /* [n_nodes] element offset of right factor               */
  const int64_t* d_off;    /* [n_nodes] element offset of dense payload              */
} hx_operand;

/* Pool offsets for an operand with the given payload kinds and ranks, in the panel order
 * hx_assemble uses: left factors grouped by row cluster, right factors by column
 * cluster, then the dense leaves.  The factors of the low-rank leaves of one block
 * column (row) are then adjacent -- one column-major |sigma| x sum(k) matrix -- which the
 * planner exploits to stack cores panel-wise.  Any other layout stays valid input to
 * hx_plan_create (only slower).  Replaces the leaf-by-leaf storage of HMatrix.data
 * (pkg/src/hmat/hmatrix.py:48-65) for the device pools. */
int hx_operand_layout(const hx_tree* tree, const int8_t* payload, const int32_t* rank,
                      int64_t* u_off, int64_t* v_off, int64_t* d_off, int64_t* pool_elems);

/* HMX1 operator files (reference format pkg/src/hmat/hmatrix.py:9-24), read and written
 * straight from / into a packed pool with the directory above.
 * hx_hmx1_write replaces save_hmatrix (hmatrix.py:338-361): records in ascending node id,
 * row-major payloads; `fingerprint` = sha256 of the block-tree dump (tree_fingerprint,
 * hmatrix.py:334-335); `degraded` [n_nodes] may be NULL.
 * hx_hmx1_scan + hx_hmx1_read replace load_hmatrix (hmatrix.py:364-388): the scan checks
 * the header (HX_EINVAL with the reference's messages: "not an H-matrix file",
 * "unsupported version V", "dimension mismatch: file N, tree M", "block tree does not match
 * the stored operator"), every record against the tree, and returns per node the payload
 * kind (1 low rank, 2 dense), rank, degraded flag and payload file position; the caller
 * lays the pool out (hx_operand_layout) and hx_hmx1_read fills it. */
int hx_hmx1_write(const char* path, const hx_tree* tree, int64_t n, const uint8_t* fingerprint,
                  const hx_operand* op, const int8_t* degraded, const double* pool);
int hx_hmx1_scan(const char* path, const hx_tree* tree, int64_t n, const uint8_t* fingerprint,
                 int8_t* payload, int32_t* rank, int8_t* degraded, int64_t* pos);
int hx_hmx1_read(const char* path, const hx_tree* tree, const hx_operand* op,
                 const int64_t* pos, double* pool);

typedef struct hx_plan hx_plan;
typedef struct hx_ctx hx_ctx;

typedef struct hx_plan_info {
  int64_t n_out;            /* output leaves in this plan (far + near)             */
  int64_t n_far, n_near;
  int64_t n_terms_real;     /* terms created by the restrict descent (logged)      */
  int64_t n_terms_expand;   /* terms created by expanding pending pairs at far leaves */
  int64_t n_dxd;            /* dense x dense products                              */
  int64_t created[3];       /* real-descent terms by kind: FF, FX, XF              */
  int64_t mat_terms, mat_tiles, mat_groups;
  int64_t core_terms, core_tiles;
  int64_t fac_terms, fac_tiles;
  int64_t core_elems, term_elems, tile_elems;
  int64_t max_out_dim;      /* largest output block side                           */
  int64_t n_xgroups;        /* terms batched by their shared H-block X             */
  int64_t gather_elems, gather_jobs;
  double flops_form, bytes_form;   /* canonical model term formation   */
  double flops_near, bytes_near;   /* canonical model near leaves                    */
} hx_plan_info;

/* ---- planning (CPU only; no GPU needed) ---------------------------------------------
 * leaf_mask (nullable, [n_nodes]): nonzero for output leaves this process owns; terms
 * are only built for blocks on the root path of an owned leaf (multi-GPU partition).
 * tile: CTA tile side (32 or 64).
 * flags: HX_PLAN_DEFER leaves the per-batch core / X G work lists to hx_product, which
 * fills them batch by batch while the device runs the previous batches; the caller's
 * tree / operand arrays must then stay alive until hx_product returns.
 * HX_PLAN_LOG keeps the restrict log for hx_plan_term_log (parity tests).
 * HX_PLAN_IMPLICIT(l): far leaves with min(m, n) >= 2^l are never materialized; hx_product
 * sketches them straight from their terms (range pass Z = R^T Omega, Y = L Z; co-range
 * W = L^T Q, B^T = R W) and estimates the unsampled tail from extra probe columns.  The
 * route the canonical work model prices as "sketch".
 * HX_PLAN_TRAD(c): the traditional-mode product (hmult_traditional, multiply.py:259-263):
 * every pending pair of a far leaf is converted to low rank on its own -- c = 1 by the
 * hierarchical agglomeration (converter "hier-approx", multiply.py:140-189), c = 2 by one
 * best approximation of the pair product (converter "dense-svd") -- and each far leaf is
 * the norm-sorted pairwise truncated sum of its terms (fast_truncate_sum). */
#define HX_PLAN_DEFER 1
#define HX_PLAN_LOG 2
#define HX_PLAN_TRAD_SHIFT 4
#define HX_PLAN_TRAD(c) ((int)(c) << HX_PLAN_TRAD_SHIFT)
#define HX_PLAN_IMPLICIT_SHIFT 8
#define HX_PLAN_IMPLICIT(l) ((int)(l) << HX_PLAN_IMPLICIT_SHIFT)
int hx_plan_create(const hx_tree* tree, const hx_operand* a, const hx_operand* b,
                   const uint8_t* leaf_mask, int tile, int flags, hx_plan** out);
int hx_plan_info_get(const hx_plan* plan, hx_plan_info* info);
/* Per output leaf (plan order): block id, kind (1 far / 2 near), m, n, stacked rank K,
 * dense-pair flops F_DD and elements E_DD (canonical model inputs). Any pointer may be
 * NULL. */
int hx_plan_leaves(const hx_plan* plan, int32_t* ids, int8_t* kind, int32_t* m,
                   int32_t* n, int64_t* stacked_rank, double* f_dd, double* e_dd);
/* Terms created by the restrict descent, in creation order: creation block, kind
 * (0 FF, 1 FX, 2 XF), A node, B node, rank — the instrumented replay of
 * sumexpr.py:146-151. */
int hx_plan_term_log(const hx_plan* plan, int32_t* block, int8_t* kind, int32_t* a_node,
                     int32_t* b_node, int32_t* rank);
void hx_plan_free(hx_plan* plan);
/* Tensor-core work of the core, factor and materialization batches: flops[0..2] as issued
 * (full tiles, k padded to 4), flops[3..5] useful (term extents, exact k). */
int hx_plan_mma_flops(hx_plan* plan, double* flops);

/* ---- device context ----------------------------------------------------------------- */
int hx_ctx_create(int device, hx_ctx** out);
/* which: 0 = A, 1 = B.  host != NULL: copy n_elems doubles from host memory.
 * host == NULL and device != NULL: attach an existing device pool (not owned). */
int hx_ctx_operand(hx_ctx* ctx, int which, const double* host, const double* device,
                   int64_t n_elems);
/* Reuse A's pool for B (A is B). */
int hx_ctx_operand_alias(hx_ctx* ctx);

typedef struct hx_product_cfg {
  int32_t policy;        /* 0 EpsRank, 1 FixedRank (lowrank.py:57-72)               */
  double eps;            /* EpsRank.eps (already clamped by the caller)             */
  int32_t k_max;         /* FixedRank.k_max                                         */
  int32_t tag;           /* 0 aca, 1 bilanczos, 2 randomized, 3 dense-svd: 0-2 run the
                          * reference's matrix-free schemes on the implicit sums
                          * (compressors.py:162-428), 3 the sketch + SVD route      */
  uint64_t seed;         /* CompressorKind.seed                                     */
  int32_t sketch0;       /* initial sketch width (0 = default)                      */
  int32_t oversample;    /* minimum sketch oversampling (0 = default 6)             */
  int32_t q;             /* CompressorKind.q: randomized subspace iterations        */
} hx_product_cfg;

typedef struct hx_product_stats {
  double ms_total;       /* CUDA-event time of the whole product on the device      */
  double ms_form, ms_mat, ms_recompress;
  int64_t far_leaves, near_leaves, degraded_blocks, max_far_rank;
  int64_t matvec_count;  /* the reference's CountingMap total (compressors.py:88-119):
                          * dense-svd n per far block, the matrix-free tags the rows,
                          * columns and matvecs their iterations applied             */
  int64_t sketch_rounds;
  int64_t launches;      /* kernels launched by this call                           */
  int64_t out_elems;     /* doubles in the packed result                            */
  double fro2_total;     /* sum of squared Frobenius norms of all output blocks     */
  double dom_kernel_ms;  /* summed device time of the materialization launches      */
  double ms_upload;      /* H2D of the plan's work lists (inside ms_total)          */
  double t_marks[4];     /* start, formation end, materialization end, end: ms after the
                          * device epoch (hx_timeline_epoch), -1 without an epoch    */
  int64_t sketch_cols;   /* operator columns the dense-svd sketch route applied     */
} hx_product_stats;

/* Records the device epoch the t_marks of later products are measured from. */
int hx_timeline_epoch(void);

int hx_product(hx_ctx* ctx, hx_plan* plan, const hx_product_cfg* cfg,
               hx_product_stats* stats);
/* Per output leaf (plan order): rank (-1 near), degraded flag, element offset of the
 * leaf's payload in the packed result (left m x r then right n x r, or dense m x n,
 * column-major). */
int hx_result_layout(hx_ctx* ctx, int32_t* rank, int8_t* degraded, int64_t* offset);
int hx_result_download(hx_ctx* ctx, double* host, int64_t n_elems);

/* ---- GPU operand assembly (assemble_hmatrix, hmatrix.py:97-118) ----------------------
 * points: [n x dim] row-major in TREE order (points[perm]); kernel: 0 exp(-r),
 * 1 exp(-r/0.5), 2 exp(-r^2/0.1), 3 1/(r+h).  Far leaves by partially pivoted ACA at eps
 * (compressors.py:162-247, with its eps/2 SVD recompression :245-246; a block whose ACA
 * cannot certify convergence falls back to dense storage and is flagged), near leaves
 * dense.  The packed pool (hx_operand layout) is allocated on the device and returned in
 * *pool_dev; per-node payload/rank/offsets/degraded flags are written to host arrays of
 * length tree->n_nodes.  Free the pool with hx_pool_free. */
int hx_assemble(hx_ctx* ctx, const hx_tree* tree, const double* points, int dim, int kernel,
                double h, double eps, int8_t* payload, int32_t* rank, int64_t* u_off,
                int64_t* v_off, int64_t* d_off, int8_t* degraded, double** pool_dev,
                int64_t* pool_elems);
/* Copy n_elems doubles of a library-allocated device pool to host memory (or to another
 * device buffer: the copy direction is inferred from the pointers). */
int hx_pool_download(hx_ctx* ctx, const double* pool_dev, double* host, int64_t n_elems);
int hx_pool_free(hx_ctx* ctx, double* pool_dev);

/* Diagnostics: batched Householder QR of n_jobs column-major panels (p[i] x q[i], q <= p,
 * concatenated in X, overwritten by the explicit Q; R gets the q x q factors), through the
 * same dispatch as the recompression (register / warp / CTA kernels, TSQR for tall panels). */
int hx_debug_qr(int n_jobs, const int32_t* p, const int32_t* q, double* X, double* R);
/* Diagnostics: run the grouped DMMA GEMM kernel on host data (Term / Tile / Group records
 * of paper_1805_08998_b200/csrc/hx_types.h; host_bufs/buf_elems: 10 buffer slots, copied to
 * the device and back).  tile = 32 or 64, or -64 for the 64-tile kernel configured for
 * short-K batches (term formation).  Used by the kernel-level parity tests. */
int hx_debug_gemm(int tile, const void* terms, int64_t n_terms, const void* tiles,
                  int64_t n_tiles, const void* groups, int64_t n_groups,
                  double* const* host_bufs, const int64_t* buf_elems, double* sumsq,
                  int64_t n_sumsq);

/* Diagnostics: numpy's default_rng(seed).standard_normal(n) stream, seed = seed_hi * 2^64 +
 * seed_lo, generated on the host (device < 0) or by the device generator the matrix-free
 * compressors use (the reference's per-block streams, multiply.py:61-63). */
int hx_np_normals(uint64_t seed_lo, uint64_t seed_hi, int64_t n, double* out, int device);
/* Diagnostics: one dense column-major m x n block through the matrix-free compressor route
 * of hx_product (tag 0 aca, 1 bilanczos, 2 randomized: compressors.py:162-428, with the
 * per-block stream default_rng((seed << 24) ^ node)); left / right get rank columns
 * (room for min(m, n)); info = {rank, degraded, matvec count}. */
int hx_debug_compress(int tag, int policy, double eps, int k_max, int q, uint64_t seed,
                      int32_t node, int m, int n, const double* A, double* left,
                      double* right, int32_t* info);

int hx_ctx_synchronize(hx_ctx* ctx);
/* Device memory available to the context (free + the workspace it already holds). */
int hx_ctx_mem_info(hx_ctx* ctx, int64_t* free_bytes, int64_t* total_bytes);
/* Device memory the context holds as reusable workspace. */
int64_t hx_ctx_held_bytes(hx_ctx* ctx);
/* Attach the operand pools of src (same device) to dst without copying, so that two
 * contexts -- two streams -- can run products (chunks) concurrently. */
int hx_ctx_operand_share(hx_ctx* dst, hx_ctx* src);
/* Page-locked host memory for the caller's result blocks (from the library's reuse cache;
 * hx_host_free returns it) and registration of caller-owned pools for fast uploads. */
void* hx_host_alloc(int64_t bytes);
void hx_host_free(void* p, int64_t bytes);
int hx_host_register(void* p, int64_t bytes);
int hx_host_unregister(void* p);
/* Release the product workspace (work lists, term/tile buffers, results not yet
 * downloaded); operand pools stay attached. */
int hx_ctx_trim(hx_ctx* ctx);
/* Forget the per-size-class rank hints that narrow the first sketch of later chunks of
 * one product (called at the start of every product). */
int hx_ctx_reset_hints(hx_ctx* ctx);

/* Y = M X (transpose = 0) or M^T X (transpose = 1) for the H-matrix attached in operand
 * slot `which` (0 or 1) of the context: X and Y are host n x s column-major blocks in
 * tree ordering.  Replaces hmat_vec / hmat_vec_transpose / _node_matmat
 * (pkg/src/hmat/hmatrix.py:138-211) for a block of s probe vectors at once; used to
 * estimate ||C - A B|| of products too large to materialize. */
int hx_hmatvec(hx_ctx* ctx, const hx_tree* tree, const hx_operand* op, int which,
               int transpose, const double* X, double* Y, int s);
void hx_ctx_free(hx_ctx* ctx);

int hx_last_error(char* buf, size_t len);
int hx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HX_H */
