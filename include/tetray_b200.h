/*
 * tetray_b200.h -- C ABI of libtetray_b200.so, the B200-native replacement
 * for the tetray render hot path (arXiv 1908.01906 reference).
 *
 * The reference's only FFI on this path is the numba call
 *   _kernels.render_frame(<49 positional args>)      pkg/src/tetray/_kernels.py:312-322
 * assembled by render()                              pkg/src/tetray/render.py:183-193
 * plus the batched point query
 *   _kernels.field_at_many(pts, <mesh args>)         pkg/src/tetray/_kernels.py:157-170
 * and the host-side producers of its inputs (mesh.py:246-260, partitions.py:73-128,
 * traversal.py:82-99, transfer.py:95-167).  This header replaces each of them;
 * the mapping is given per entry point.  All entry points return 0 on success
 * and a nonzero TR_E* code on failure, with tr_last_error() describing it; they
 * never abort.  No torch types appear here: device buffers are plain pointers
 * (owned by the caller -- in the Python host layer, torch tensors).
 *
 * Device data layout:
 *   TrTetRecord[T]   128 B/tet: inverse edge matrix, origin, 4 field values
 *   TrPNode[]        64 B BVH2 nodes over padded tet boxes, f32 child boxes
 *   TrPLeaf[]        32 B leaf headers: exclusive box + id range
 *   uint32 leaf ids  ascending per leaf (lowest-index-first scan)
 *   TrBNode[]        112 B BVH2 nodes over partition boxes, f64 child boxes
 */
#ifndef TETRAY_B200_H
#define TETRAY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TR_OK 0
#define TR_EINVAL 1   /* bad argument */
#define TR_ECUDA 2    /* CUDA runtime error */
#define TR_ENOMEM 3   /* host allocation failure */
#define TR_ESTATE 4   /* object in the wrong state */

/* ------------------------------------------------------------ layouts */

/* One tetrahedron, 128 B (one L2 line).  inv/orig are the reference's
 * MeshSampler.tet_inv / tet_orig (mesh.py:251-254) bit for bit; f[i] is
 * field[tets[t,i]] for vertex-centered data, f[0] = field[t] for cell data. */
typedef struct TrTetRecord {
    double inv[9];
    double orig[3];
    double f[4];
} TrTetRecord;

/* Point-location BVH2 node: both child boxes (f32, rounded outward from the
 * f64 padded tet boxes of mesh.py:248-250), child links and the minimum tet
 * id below each child.  child >= 0: node index; child < 0: leaf ~child;
 * child == INT32_MIN: no child. */
typedef struct TrPNode {
    float lo0[3], hi0[3], lo1[3], hi1[3];
    int32_t child[2];
    uint32_t minid[2];
} TrPNode;

/* Leaf header, 64 B.  ex_lo/ex_hi: the leaf's EXCLUSIVE box (rounded
 * inward to f32): no other leaf's box meets its interior, so a point
 * strictly inside it can only be contained by this leaf's tets.
 * walk: the leaf walk table (tr_leaf_walk; all zero = no walk, the leaf is
 * scanned in id order).  For leaf-local tet i < 8, the 16-bit entry
 * (walk[i / 2] >> (16 * (i % 2))): bits [3f, 3f+3) = the leaf-local tet
 * across the face opposite vertex f (i itself: none in the leaf); bit 12 =
 * CERTIFIED: a point whose barycentrics in tet i are all >= TR_WALK_TAU lies
 * outside every lower-id tet of the leaf with the reference's -1e-9 slack
 * (K:128), so tet i is the lowest-index containing tet (K:119) without
 * testing them.  walk[4]: bits 0-2 = the walk's first tet (the largest),
 * bit 31 = table valid. */
typedef struct TrPLeaf {
    float ex_lo[3], ex_hi[3];
    uint32_t start, count;
    uint32_t walk[8];
} TrPLeaf;

/* The walk's certification margin on the barycentrics (tr_leaf_walk). */
#define TR_WALK_TAU 1e-6

/* Walk-start predictor of a leaf (48 B): approximate barycentrics l1..l3 of
 * the leaf's first tet, l_r ~ row[r][0]*(x - ex_lo[0]) + row[r][1]*(y - ex_lo[1])
 * + row[r][2]*(z - ex_lo[2]) + row[r][3], in f32.  The march evaluates them
 * (no record load) and starts the walk at the first tet's neighbour across
 * the face it predicts the point is beyond; a wrong guess only costs a walk
 * step -- acceptance is always the exact test + certificate. */
typedef struct TrLeafPred {
    float row[3][4];
} TrLeafPred;

/* Partition BVH2 node: f64 child boxes (exact unions of partition boxes,
 * so node pruning is conservative for the exact f64 slab test).
 * child >= 0: node; child < 0: partition ~child; INT32_MIN: none. */
typedef struct TrBNode {
    double box[2][6]; /* per child: lo x,y,z then hi x,y,z (48 B, 16-B aligned) */
    int32_t child[2];
    int32_t pad[2];
} TrBNode;

/* Partition BSP node (pre-order; the left child is the next node).
 * info >= 0: split on axis info & 3 at `split`, right child info >> 2.
 * info <  0: leaf holding aux partitions leaf_pids[~info ..]. */
typedef struct TrKNode {
    double split;
    int32_t info;
    int32_t aux;
} TrKNode;

/* ------------------------------------------------- host-side builders */
/* Opaque host object holding variable-size build results. */
typedef struct TrHostBuf TrHostBuf;

/* KD partitions, replacing partitions.build_partitions (partitions.py:73-128)
 * with the reference's exact split/median/straddle/leaf semantics.
 * Result arrays via tr_kd_* getters below. */
int tr_kd_build(int64_t n_vertices, const double *vertices, int64_t n_tets, const int64_t *tets,
                const double *field, int32_t centering, const double *mesh_lo,
                const double *mesh_hi, int64_t max_leaf_elements, int64_t max_depth,
                TrHostBuf **out);
/* The same KD partitions in closed form for the synthetic N^3-cube mesh
 * (mesh.py:147-231: five tets per cube, vertex field 0 = ramp, 1 = radial),
 * without the mesh arrays (1e9-tet scenes).  with_ids (N <= 256) also lists
 * the element ids; otherwise tr_kd_sizes reports 0 ids. */
int tr_kd_build_grid(int64_t n, int32_t field, int64_t max_leaf_elements, int64_t max_depth,
                     int32_t with_ids, TrHostBuf **out);
/* sizes: [0] = n_parts, [1] = total element ids */
int tr_kd_sizes(const TrHostBuf *kd, int64_t *sizes2);
/* offsets[n_parts+1], ids[total], leaf_lo/hi[n_parts*3] (KD leaf boxes),
 * lo/hi[n_parts*3] (refined bounds, partitions.py:61-70), vrange[n_parts*2] */
int tr_kd_copy(const TrHostBuf *kd, int64_t *offsets, int64_t *ids, double *leaf_lo,
               double *leaf_hi, double *lo, double *hi, double *vrange);

/* Point-location BVH over padded tet boxes (replaces MeshSampler's BVH,
 * mesh.py:248-250 / bvh.py:41-98; any conservative structure gives the
 * reference's lowest-index result). */
int tr_pbvh_build(int64_t n_tets, const double *box_lo, const double *box_hi, int32_t leaf_max,
                  TrHostBuf **out);
/* sizes: [0] = nodes, [1] = leaves, [2] = leaf ids, [3] = grid cells */
int tr_pbvh_sizes(const TrHostBuf *b, int64_t *sizes4);
int tr_pbvh_copy(const TrHostBuf *b, TrPNode *nodes, TrPLeaf *leaves, uint32_t *ids);
/* Fill the walk tables of leaves[0, n_leaves) (in place) from the mesh:
 * rec_ids[k] = tet id of record k (NULL: k), vertices (V,3), tets (T,4).
 * Face neighbours are matched by shared vertex ids; the CERTIFIED bit of
 * tet i is set only when, for every lower-id tet j of the leaf, a face plane
 * of j separates tet i shrunk to barycentrics >= TR_WALK_TAU from j by more
 * than the 1e-9 slack plus a 1e-8 margin, or a face plane of i separates j
 * inflated by that slack from the shrunk tet (checked in long double at the
 * shrunk/inflated vertices; leaves whose coordinates are too large for
 * those margins to cover the device's rounding get no certificates).  Leaves
 * of more than 8 tets get no table. */
int tr_leaf_walk(int64_t n_leaves, TrPLeaf *leaves, const uint32_t *rec_ids,
                 const double *vertices, const int64_t *tets, TrLeafPred *pred);
/* pred (n_leaves, may be NULL): the walk-start predictor of each leaf,
 * relative to its ex_lo (set the exclusive boxes first). */
/* The two predictors of tr_grid_scene_build's cubes (even, odd parity), for
 * TrDeviceScene.pred_class (interior cubes; boundary cubes differ by the pad). */
int tr_grid_walk_pred(double pad, TrLeafPred *pred2, uint32_t *walk16);
/* walk16 (may be NULL): the two cubes' TrPLeaf.walk tables, 2 x 8 u32. */
/* Uniform-grid leaf index: cell (x,y,z) -> leaf whose exclusive box covers
 * most of it (-1: none).  cell = floor((p - org) * scale), row-major x,y,z. */
int tr_pbvh_grid(const TrHostBuf *b, int32_t *dims3, double *org3, double *scale3,
                 int32_t *cells);

/* Mean fraction of a grid cell covered by its candidate leaf's exclusive box
 * (1 for the generator's regular meshes; low for unstructured meshes). */
double tr_pbvh_coverage(const TrHostBuf *b);
/* Cell candidate lists (the exact point-location path for unstructured
 * meshes): a grid refined `refine` times per axis over the point BVH's grid;
 * cell c lists the records (leaf order) whose padded tet boxes (box_lo/hi,
 * by tet id) meet it, in ascending tet id; off[c] bit 31 marks cells over
 * max_list entries (BVH descent there).  tbox: 8 floats per record = its
 * padded box rounded outward (lo xyz, hi xyz, 2 pad). */
int tr_cells_build(const TrHostBuf *pbvh, const double *box_lo, const double *box_hi,
                   int32_t refine, int32_t max_list, TrHostBuf **out);
/* sizes: [0] cells, [1] list entries, [2] records */
int tr_cells_sizes(const TrHostBuf *cells, int64_t *sizes3);
int tr_cells_copy(const TrHostBuf *cells, int32_t *dims3, double *org3, double *scale3,
                  uint32_t *off, uint32_t *recs, float *tbox);

/* Partition BVH (replaces traversal.build_partition_bvh, traversal.py:82-91). */
int tr_bbvh_build(int64_t n_parts, const double *lo, const double *hi, TrHostBuf **out);
int tr_bbvh_sizes(const TrHostBuf *b, int64_t *n_nodes);
int tr_bbvh_copy(const TrHostBuf *b, TrBNode *nodes);
/* Per-epoch subtree activity: out[node] bit c = child c reaches an active partition. */
int tr_bbvh_activity(const TrHostBuf *b, const uint8_t *active, uint8_t *out);
/* Same from a node array (no host object needed). */
int tr_bnodes_activity(int64_t n_nodes, const TrBNode *nodes, const uint8_t *active,
                       uint8_t *out);

/* Axis-aligned BSP over the partition boxes (greedy separating planes; the
 * KD split planes for KD partitions): front-to-back partition enumeration
 * for the trace pass.  root6 = union box (lo xyz, hi xyz). */
int tr_kbsp_build(int64_t n_parts, const double *lo, const double *hi, TrHostBuf **out);
int tr_kbsp_sizes(const TrHostBuf *b, int64_t *sizes2);
int tr_kbsp_copy(const TrHostBuf *b, TrKNode *nodes, int32_t *leaf_pids, double *root6);
/* Per-epoch: out[node] = 1 if the subtree holds an active partition. */
int tr_knodes_activity(int64_t n_nodes, const TrKNode *nodes, const int32_t *leaf_pids,
                       const uint8_t *active, uint8_t *out);

void tr_host_free(TrHostBuf *b);

/* Pack tet records (host, OpenMP). inv/orig exactly as MeshSampler computes
 * them; out[k] holds tet order[k] (order = point-BVH leaf order; NULL: k). */
int tr_pack_tets(int64_t n_tets, const int64_t *tets, const double *tet_orig,
                 const double *tet_inv, const double *field, int32_t centering,
                 const uint32_t *order, TrTetRecord *out);
/* Padded tet boxes (mesh.py:248-250: vertex min/max -+ pad), OpenMP. */
int tr_tet_boxes(int64_t n_tets, const double *vertices, const int64_t *tets, double pad,
                 double *lo, double *hi);

/* Transfer-function partition metadata (transfer.py:95-141): per partition
 * max opacity, raw variance (numpy reduction order reproduced), normalized
 * sigma, active flag. */
int tr_tf_meta(int64_t n_parts, const double *vrange, const double *tf_table, int64_t n_tf,
               double tf_lo, double tf_hi, double *max_opacity, double *raw_variance,
               double *sigma, uint8_t *active);

/* The same metadata on the GPU (csrc/meta.cu, one thread per partition,
 * numpy's reduction order kept: identical results).  All pointers are device
 * pointers; sigma / active may be NULL.  Synchronizes the stream. */
int tr_tf_meta_device(int64_t n_parts, const double *vrange, const double *tf_table, int64_t n_tf,
                      double tf_lo, double tf_hi, double *max_opacity, double *raw_variance,
                      double *sigma, uint8_t *active, void *stream);

/* The epoch's step arrays on the device (device pointers): step[n] and
 * step_ratio[n][2] from sigma[n] with the restated glibc pow; *inexact is set
 * (to 1) if any entry fell outside the restated path -- the caller must then
 * use tr_epoch_steps on the host (the bench/render path checks the domain on
 * the host first, so no read-back is needed). */
int tr_epoch_steps_device(int64_t n, const double *sigma, double s1, double s2, double p,
                          double *step, double *step_ratio, int32_t *inexact, void *stream);

/* step_size (K:20-22) per partition on the host with glibc pow, so adaptive
 * steps are bit-identical to the reference's. */
int tr_step_sizes(int64_t n, const double *sigma, double s1, double s2, double p, double *out);
double tr_step_size(double s1, double s2, double p, double sigma);
/* Both epoch step arrays at once: step[n] and step_ratio[n][2] = {step,
 * step / s1} (opacity_correction's exponent, K:27); either may be NULL. */
int tr_epoch_steps(int64_t n, const double *sigma, double s1, double s2, double p, double *step,
                   double *step_ratio);
double tr_opacity_correction(double alpha, double s, double s1);

/* glibc pow restated (csrc/glibc_pow.cuh): 1 if the tables were found in the
 * installed libm at build time (the device then evaluates the per-sample
 * opacity correction bit-identically to the reference). */
int tr_pow_glibc_available(void);
/* Host evaluation of the restatement; *exact = 0 outside the restated path. */
double tr_pow_glibc_host(double x, double y, int32_t *exact);
/* Device evaluation over n argument pairs (device pointers). */
int tr_pow_glibc_batch(int64_t n, const double *x, const double *y, double *out, void *stream);

/* ------------------------------------------------- device entry points */

/* Device-resident scene (device pointers, owned by the caller). */
typedef struct TrDeviceScene {
    const TrTetRecord *tets;
    const TrPNode *pnodes;
    const TrPLeaf *pleaves;
    const uint32_t *pleaf_ids;  /* tet id of each record; NULL: record k is tet k */
    int64_t n_tets, n_pnodes, n_pleaves;
    int32_t centering;
    int32_t pad0;
    const TrBNode *bnodes;
    const double *part_lo; /* (P,3) refined partition bounds */
    const double *part_hi;
    int64_t n_parts, n_bnodes;
    double mesh_lo[3], mesh_hi[3];
    const int32_t *pgrid;  /* tr_pbvh_grid cells */
    const TrPLeaf *pgrid_leaf; /* per cell: copy of its candidate leaf's header (empty box: none) */
    int32_t gdim[3];
    int32_t pad1;
    double gorg[3], gscale[3];
    const TrKNode *knodes; /* tr_kbsp_* (NULL: trace with the partition BVH) */
    const int32_t *kleaf_pids;
    int64_t n_knodes;
    double kroot[6];
    /* cell candidate lists (tr_cells_*; NULL: none -- BVH descent instead) */
    const uint32_t *cell_off;
    const uint32_t *cell_recs;
    const float *tbox;
    int32_t cdim[3];
    int32_t cells_first;   /* 1: skip the exclusive-leaf grid (it rarely proves a point) */
    double corg[3], cscale[3];
    /* walk-start predictors: per grid cell (a copy of its leaf's, like
     * pgrid_leaf), or -- pgrid_pred NULL, pred_classes 2 -- one per cube
     * parity (tr_grid_scene_build's scenes); neither: no prediction */
    const TrLeafPred *pgrid_pred;
    int32_t pred_classes;
    int32_t pad2;
    TrLeafPred pred_class[2];
    /* analytic leaves of tr_grid_scene_build's n^3 cube grids (grid_n > 0):
     * the march computes a sample's cube, its exclusive box and record range
     * from the coordinates (the layout tr_grid_scene_build wrote; grid_brick:
     * 8^3-cube brick order) and walks it with class_walk (device, 2 x 8 u32:
     * the TrPLeaf.walk of an even / odd cube) -- no leaf header load */
    int64_t grid_n;
    double grid_pad;
    int32_t grid_brick;
    int32_t pad3;
    const uint32_t *class_walk;
} TrDeviceScene;

/* One metadata epoch (scene.meta_state(), scene.py:48-50 / 78-82), device pointers. */
typedef struct TrEpoch {
    const uint8_t *active;       /* (P,) */
    const uint8_t *bnode_active; /* (n_bnodes,) from tr_bbvh_activity */
    const double *step;          /* (P,) host step_size; only read in mode 2 */
    const double *tf_table;      /* (n_tf, 4) */
    int64_t n_tf;
    double tf_lo, tf_hi;
    const uint8_t *knode_active; /* (n_knodes,) from tr_knodes_activity, or NULL */
    const double *step_ratio;    /* (P,2) interleaved {step, step / s1} (opacity_correction's
                                    exponent, K:27); only read in mode 2 */
    const int32_t *inexact;      /* device word, nonzero if a device step was inexact (entries
                                    NaN; render() raises); NULL when the host made the steps */
} TrEpoch;

/* One metadata epoch in one call (R:169; scene.py:78-82): packs sigma, the TF
 * table and the activity bits into the page-locked host_buf, copies them to
 * dev_buf (tr_epoch_bytes(...) bytes) on `stream` and computes the per-partition
 * steps there (steps_on_device: tr_epoch_steps_device, the caller having
 * checked the restated pow domain; else tr_epoch_steps on the host and the
 * whole buffer is copied).  Fills `out` with the device section pointers. */
int64_t tr_epoch_bytes(int64_t n_parts, int64_t n_tf, int64_t n_bnodes, int64_t n_knodes);
int tr_epoch_upload(int64_t n_parts, const double *sigma, const uint8_t *active,
                    const uint8_t *bnode_active, int64_t n_bnodes, const uint8_t *knode_active,
                    int64_t n_knodes, const double *tf_table, int64_t n_tf, double tf_lo,
                    double tf_hi, double s1, double s2, double p, int32_t steps_on_device,
                    void *host_buf, void *dev_buf, int64_t buf_bytes, TrEpoch *out,
                    int64_t *h2d_bytes, void *stream);

/* tr_epoch_upload's arguments as one struct (a binding builds it once per
 * epoch and re-uploads with a single call: tr_epoch_upload_s, or inside
 * tr_render_sync). */
typedef struct TrEpochUpload {
    int64_t n_parts;
    const double *sigma;
    const uint8_t *active, *bnode_active, *knode_active;
    int64_t n_bnodes, n_knodes;
    const double *tf_table;
    int64_t n_tf;
    double tf_lo, tf_hi, s1, s2, p;
    int32_t steps_on_device;
    int32_t packed;            /* host_buf already holds this epoch's sections (an
                                  earlier call packed them; the arrays are immutable):
                                  re-upload without packing -- with steps_on_device,
                                  ONE kernel reads the page-locked block over PCIe
                                  and writes the sections and the steps */
    void *host_buf, *dev_buf;
    int64_t buf_bytes;
} TrEpochUpload;
int tr_epoch_upload_s(const TrEpochUpload *u, TrEpoch *out, int64_t *h2d_bytes, void *stream);

/* Frame parameters: render_frame's scalars (K:313-316, R:183-188). */
typedef struct TrFrame {
    double cam_pos[3], cam_right[3], cam_up[3], cam_fwd[3];
    double tan_half, aspect;
    int64_t width, height;
    int32_t jitter, mode; /* mode: 0 reference, 1 skip, 2 skip-adaptive (R:27) */
    double s1, term, eps;
    double bg[4];
    int32_t track_ppart;
    int32_t shard_rank, shard_count; /* pixel tiles t with t % count == rank */
    int32_t compact;                 /* 1: write tile-major compact slots (multi-GPU) */
    int32_t flags;                   /* TR_FLAG_* */
    int32_t pad0;
} TrFrame;

#define TR_FLAG_PAIR_SCAN 64   /* leaf scan two records at a time (tuning; default: one at a time) */
#define TR_FLAG_REG_STATE 128  /* march with the per-ray state in registers (tuning; default: shared memory) */
#define TR_FLAG_TILE_TIMING 0x10000 /* trace pass: SM cycles per 32-ray tile into the kernel stats (profiling) */
#define TR_FLAG_NO_CELLS 0x20000 /* ignore the cell candidate lists: BVH descent instead (testing) */
#define TR_FLAG_NO_BG_WRITER 0x40000 /* host framebuffer: trace writes background pixels itself (testing) */
/* flags bits 20-22: trace CTAs per SM (0 = occupancy maximum; tuning) */
#define TR_FLAG_NO_CAND 0x800000 /* modes 1/2: intervals by the per-ray BSP walk, not the candidate raster (testing) */
#define TR_FLAG_FORCE_CAND 0x1000000 /* the candidate raster also above 1M pixels (default there: the BSP walk) */
#define TR_FLAG_NO_WALK 0x2000000 /* exclusive leaves scanned in id order, not walked (testing) */
#define TR_FLAG_NO_PRED 0x4000000 /* leaf walks start at the first tet, no predictor (testing) */
#define TR_FLAG_NO_ANALYTIC 0x8000000 /* grid scenes: load leaf headers, not the analytic layout (testing) */
#define TR_FLAG_NO_GRID 2      /* disable the uniform-grid leaf index (testing) */
#define TR_FLAG_STATS 4        /* count kernel events (tr_kernel_stats); slows the frame */
#define TR_FLAG_NO_BSP 8       /* where the BSP walk runs (TR_FLAG_NO_CAND, lists > 48): the partition BVH instead */
/* flags bits 8-11: log2 of the lanes that march one ray together (0 = chosen
 * per ray chunk on the device, 4 or 16, from the rays' sample counts);
 * bits 12-13: register budget of the G = 4 kernel as minimum resident CTAs
 * per SM (0: 3, 1: 4, 2: 2, 3: 3); bits 14-15: CTAs per SM actually
 * launched (0: as many as fit).  Tuning knobs only:
 * every setting renders the same frame. */

/* Outputs (device pointers).  Image layout: rgba (H,W,4) f64, samples (H,W)
 * i64, visited (H,W) i32.  Compact layout: slot-major 8x4 pixel tiles.
 * ppart (P,) u64 and totals[2] = {sum samples, sum visited} are ACCUMULATED
 * (zero them first); work[1] is a queue counter, zeroed by the call. */
typedef struct TrOutputs {
    double *rgba;
    int64_t *samples;
    int32_t *visited;
    uint64_t *ppart;
    uint64_t *totals;
    uint32_t *work;
    void *scratch;          /* interval lists (modes 1, 2); size via tr_scratch_bytes */
    int64_t scratch_bytes;  /* smaller than a frame's need => the frame runs in ray chunks */
    void *ev_march_begin;   /* optional cudaEvent_t recorded before the first march launch */
    void *ev_march_end;     /* optional cudaEvent_t recorded after the last march launch */
} TrOutputs;

/* Device address of page-locked host memory (cudaHostGetDevicePointer):
 * TrOutputs.rgba / samples may point there, so the march writes each finished
 * pixel straight into the caller's host framebuffer over PCIe while it runs
 * (render() does this; no separate device->host copy after the frame). */
int tr_host_device_pointer(void *host, void **dev);
/* Page-lock and map existing host memory (cudaHostRegister, mapped +
 * portable) and return its device address; render(distributed=True) maps one
 * node-shared result block (a /dev/shm file every rank has mapped) this way,
 * so each GPU writes its own pixel tiles into the frame rank 0 returns. */
int tr_host_register(void *host, int64_t bytes, void **dev);
int tr_host_unregister(void *host);
/* Stream-ordered memset / copy (cudaMemsetAsync, cudaMemcpyAsync with
 * cudaMemcpyDefault): the per-frame counter reset and read-back without a
 * framework dispatcher in between. */
int tr_memset_async(void *dst, int32_t value, int64_t bytes, void *stream);
int tr_copy_async(void *dst, const void *src, int64_t bytes, void *stream);

/* Scratch bytes for n_rays rays in one chunk (pass W*H rounded up to 32). */
int64_t tr_scratch_bytes(int64_t n_rays);

/* Replaces _kernels.render_frame (K:312-398). stream: cudaStream_t. */
int tr_render_frame(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                    const TrOutputs *out, void *stream);
/* render()'s whole synchronous frame in one call (R:175-204 around K:312):
 * zero the counters (out->totals: n_counters i64 = totals, work, per-partition
 * samples), tr_render_frame, copy the counters to counters_host (page-locked)
 * and the epoch's inexact word to *inexact_host (when epoch->inexact and
 * inexact_host are set), synchronize `stream`; *device_ms = the frame's
 * kernels (CUDA events).  rgba / samples land wherever `out` points. */
int tr_render_sync(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrOutputs *out, int64_t n_counters, int64_t *counters_host,
                   int32_t *inexact_host, void *stream, float *device_ms,
                   const TrEpochUpload *reupload);
/* reupload (may be NULL): copy the epoch again first (tr_epoch_upload_s into
 * the same buffers, so `epoch` stays valid). */

/* ---- Exact record-sharded (KD-brick) rendering ----
 * The partitions are grouped into n_bricks convex bricks (KD subtrees); brick
 * b's device scene holds only the tets within its box + a halo of the
 * largest step, with global tet ids (lowest-id location unchanged).  Every
 * rank traces the full interval list (the partition structures are small and
 * replicated); the ray's samples are then marched in runs: the run of
 * consecutive samples whose intervals belong to one brick is marched by that
 * brick's rank from the per-ray state the previous run left (acc rgba,
 * samples, position in the interval list), so compositing order and every
 * count are exactly the single-GPU frame's.  Mode 0's one mesh-box interval
 * is cut at the brick boxes (records keep its entry: sample k stays
 * entry + (k + phase) s1).  Rounds repeat until no ray is active; between
 * rounds the ranks exchange states.  Two exchanges: (a) SUM -- each active
 * ray was advanced by exactly one rank, so an int64 SUM all-reduce of the
 * states (zero elsewhere, zero_foreign = 1) is exact; (b) PEER (n_peers > 0)
 * -- when a run suspends, the march stores the ray's state straight into the
 * inbox of the one rank that owns its next run, over NVLink (peer_inbox: CUDA
 * IPC mappings), tagged with the round; after round 0 a rank plans only the
 * rays its inbox received in the previous round (an inbox per round parity,
 * so a round's stores never meet a reader of the round before).  Each
 * suspended ray crosses the link once, finished rays not at all, and the
 * ranks need no more than a barrier between rounds (no SUM, no host read;
 * counters[1] is then the rank's own active rays).
 * The frame must fit one ray chunk (tr_scratch_bytes(W*H)). */
typedef struct TrRayState {   /* 64 B per ray */
    double acc[4];
    int64_t samples;
    uint32_t taken;            /* samples of the ray done so far (cum space) */
    int32_t icur;              /* interval holding sample `taken` */
    uint32_t cbefore;          /* cum before interval icur */
    uint32_t stop;             /* end of the current run (set by the plan) */
    uint32_t flags;            /* 1 active, 2 done */
    uint32_t tag;              /* PEER exchange: exchange_tag of the round that wrote it + 1 */
} TrRayState;

typedef struct TrBricks {
    int32_t rank;              /* the brick this call marches */
    int32_t n_bricks;
    const int16_t *owner;      /* [n_parts] brick of each partition (device) */
    const double *brick_lo;    /* [n_bricks][3] brick boxes (device; mode 0 cut) */
    const double *brick_hi;
    TrRayState *state;         /* [rays] (device) */
    uint32_t *queue;           /* [rays] rays of this brick's current run (device) */
    uint32_t *counters;        /* [4] device: rays queued, rays active, error bits, spare */
    int32_t zero_foreign;      /* 1: zero the states of rays another brick advances (SUM exchange) */
    int32_t write_background;  /* 1: the trace writes the background pixels (one rank only) */
    /* PEER exchange (n_peers = 0: off).  exchange_tag = 256 * frame number
     * (>= 1, the same on every rank) + round; inbox = this rank's [2][rays]
     * states (device, zeroed once); peer_inbox[2 r + p] = rank r's inbox of
     * round parity p mapped here (device array of 2 n_bricks pointers). */
    uint32_t exchange_tag;
    int32_t n_peers;
    TrRayState *const *peer_inbox;
    TrRayState *inbox;
} TrBricks;

/* Trace + state init of a brick-sharded frame (any brick's scene: the
 * partition structures are global).  counters[2] bit 0: a ray needs more than
 * the stored interval list (unsupported; the caller raises). */
int tr_brick_trace(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrBricks *bricks, const TrOutputs *out, void *stream);
/* One round for brick `bricks->rank`: plan every active ray's next run, march
 * the runs that are this brick's with its scene; rays that finish write their
 * pixel, the others leave their state for the next run's brick.  counters[1]
 * = rays still active when the plan ran. */
int tr_brick_round(const TrDeviceScene *scene, const TrEpoch *epoch, const TrFrame *frame,
                   const TrBricks *bricks, const TrOutputs *out, void *stream);

/* Device build of the synthetic N^3-cube scene (mesh.py:147-231 generator,
 * vertex field 0 = ramp, 1 = radial; csrc/synth.cu) straight into HBM: n_tets
 * = 5 N^3 records, one leaf per cube (the point
 * grid is the cube grid: gorg 0, gscale 1, gdim N, pgrid_leaf = leaves) and
 * N^3 - 1 BVH nodes.  inv10: host (10,3,3) inverse edge matrices of the 5 tets
 * of an even then an odd cube (numpy's LAPACK, mesh.py:254).  pad = the box
 * pad 1e-7 * diagonal (mesh.py:249).  For BASELINE config 4 (1e9 tets). */
int tr_grid_scene_sizes(int64_t n, int64_t *n_tets, int64_t *n_leaves, int64_t *n_nodes);
int tr_grid_scene_build(int64_t n, int32_t field, double pad, const double *inv10,
                        TrTetRecord *recs, TrPLeaf *leaves, TrPNode *nodes, uint32_t *ids,
                        void *stream);
/* ids: NULL -> records in id order (pleaf_ids = NULL); else records in
 * 8^3-cube brick order and ids[k] (n_tets u32) = tet id of record k. */

/* Device build of the point-location structures of an ARBITRARY mesh
 * (csrc/pbuild.cu; replaces MeshSampler's host BVH build,
 * mesh.py:246-254 / bvh.py:41-98, and this library's host builders
 * tr_tet_boxes + tr_pbvh_build + tr_pbvh_grid + tr_cells_build): Morton
 * codes of the padded tet boxes' centres, a Karras radix tree collapsed to
 * leaves of <= leaf_max tets, bottom-up refit, exclusive boxes, the leaf grid
 * and -- when the grid's coverage is below cells_below -- the cell candidate
 * lists.  vertices (V,3) f64 and tets (T,4) i64 are DEVICE pointers; leaves
 * carry no walk tables until tr_dpb_walk.  The handle owns device buffers
 * until tr_dpb_free. */
typedef struct TrDevPointBuild TrDevPointBuild;
int tr_pbvh_build_device(int64_t n_vertices, const double *vertices, int64_t n_tets,
                         const int64_t *tets, double pad, int32_t leaf_max, double cells_below,
                         int32_t refine, int32_t max_list, void *stream, TrDevPointBuild **out);
/* sizes6: n_nodes, n_leaves, n_ids (= n_tets), grid cells, cell-list cells (0: none),
 * cell-list entries. */
int tr_dpb_sizes(const TrDevPointBuild *b, int64_t *sizes6);
int tr_dpb_grid(const TrDevPointBuild *b, int32_t *gdim3, double *gorg3, double *gscale3,
                double *coverage, int32_t *cdim3, double *corg3, double *cscale3);
/* The leaves' walk tables and walk-start predictors on the device
 * (tr_leaf_walk's tables; a CERTIFIED bit only where the orientation
 * determinants prove the separation with their error bounds, so a subset of
 * the host's long-double certificates).  vertices/tets: device pointers. */
int tr_dpb_walk(TrDevPointBuild *b, const double *vertices, const int64_t *tets, void *stream);
/* Device-to-device copy into caller buffers (any may be NULL); grid_leaf /
 * grid_pred: per grid cell, its candidate's header / predictor (an empty box
 * / zeros for -1; predictors only after tr_dpb_walk). */
int tr_dpb_copy(const TrDevPointBuild *b, TrPNode *nodes, TrPLeaf *leaves, uint32_t *ids,
                int32_t *grid, TrPLeaf *grid_leaf, TrLeafPred *grid_pred, uint32_t *cell_off,
                uint32_t *cell_recs, float *tbox, void *stream);
void tr_dpb_free(TrDevPointBuild *b);
/* tr_pack_tets on the device: every pointer a device pointer. */
int tr_pack_tets_device(int64_t n, const int64_t *tets, const double *tet_orig,
                        const double *tet_inv, const double *field, int32_t centering,
                        const uint32_t *order, TrTetRecord *out, void *stream);
/* CUDA IPC for the PEER brick exchange: a zeroed device allocation and its
 * 64-B handle; open a peer's handle (peer access enabled lazily); close; free. */
int tr_ipc_alloc(int64_t bytes, void **dptr, void *handle64);
int tr_ipc_open(const void *handle64, void **dptr);
int tr_ipc_close(void *dptr);
int tr_dev_free(void *dptr);
/* Host (pageable) -> device copy through page-locked staging (synchronous). */
int tr_upload(void *dst, const void *src, int64_t bytes, void *stream);

/* Replaces _kernels.field_at_many (K:157-170): pts (n,3) f64 device;
 * found (n,) u8, vals (n,) f64, tet (n,) i64 (may be NULL) device. */
int tr_field_at_many(const TrDeviceScene *scene, int64_t n, const double *pts, uint8_t *found,
                     double *vals, int64_t *tet, void *stream);

/* Device epilogue (csrc/epilogue.cu), device pointers:
 * imgio.framebuffer_rgb (imgio.py:36-39, 76-78): rgba (n,4) f64 -> rgb (n,3) u8;
 * imgio.heatmap_rgb (imgio.py:81-87): counts (n) i64 -> rgb (n,3) u8 through
 *   lut (256,3) u8, peak = 1 u64 of scratch (the frame maximum);
 * metrics.ssim (metrics.py:48-80): two (h,w,3) u8 images, window x window
 *   weights (f64), rec709 (3 f64), c1, c2 -> *sum = sum of the SSIM map over
 *   the valid region (divide by its size for the mean). */
int tr_quantize_rgb(const double *rgba, int64_t n_pixels, uint8_t *rgb, void *stream);
int tr_heatmap_rgb(const int64_t *counts, int64_t n_pixels, const uint8_t *lut, uint8_t *rgb,
                   uint64_t *peak, void *stream);
int tr_ssim_rgb(const uint8_t *a, const uint8_t *b, int64_t height, int64_t width, int32_t window,
                const double *weights, const double *rec709, double c1, double c2, double *sum,
                void *stream);

/* Multi-GPU merge: scatter gathered compact tiles (count ranks, slot-major)
 * into the image layout. */
int tr_scatter_tiles(int64_t width, int64_t height, int32_t shard_count,
                     const double *src_rgba, const int64_t *src_samples,
                     const int32_t *src_visited, int64_t slots_per_rank, double *rgba,
                     int64_t *samples, int32_t *visited, void *stream);

/* Number of tiles (8x4 pixels) of a frame and slots per rank. */
int64_t tr_num_tiles(int64_t width, int64_t height);
int64_t tr_slots_per_rank(int64_t width, int64_t height, int32_t shard_count);

/* Launch statistics of the last tr_render_frame on this thread:
 * [0] kernels launched, [1] grid blocks, [2] threads per block. */
int tr_last_launch(int64_t *out3);

/* Kernel event counters (up to 32) accumulated by frames rendered with
 * TR_FLAG_STATS: rounds, partial rounds, lane samples, found, grid hits,
 * descents, inline next_interval, pow calls, trace intervals, trace rays, BSP
 * overflows, BSP cells, max intervals per ray, BSP nodes, max nodes per ray,
 * max samples per ray; with TR_FLAG_TILE_TIMING the trace's cycles per
 * 32-ray tile (sum, max).  Names: _lib.STAT_NAMES.  Synchronizes. */
int tr_kernel_stats(int64_t *out, int32_t n, int32_t reset);

const char *tr_last_error(void);
int tr_abi_version(void);
/* sizeof of TrDeviceScene, TrEpoch, TrFrame, TrOutputs, TrBricks, TrRayState,
 * TrTetRecord, TrPNode, TrPLeaf, TrBNode, TrKNode (the first n; bindings check
 * their struct layouts against it). */
int tr_struct_sizes(int64_t *out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif
