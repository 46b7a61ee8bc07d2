/*
 * ccl.h -- C ABI of the B200 (sm_100a) connected-components-labeling library
 * (libccl.so), the data-parallel hot path of arxiv 1708.08180:
 *   "an optimized union-find (UF) algorithm that can label the connected
 *    components on a 2D image ... three phases: UF-based local merge, boundary
 *    analysis, and link"                              (abstract)
 *
 * Problem statement (what every entry point computes):
 *   CCL "give[s] a unique ID to each connected region in a 2D ... grid"
 *   (PAPER.md:24).  Input "Image I of size N x M" -- here H rows
 *   (the paper's M) by W columns (the paper's N = imgWidth), row-major, raster
 *   index idx(x,y) = y*W + x.  A pixel is foreground iff its
 *   byte is nonzero (reading R1; ccl_label_threshold_async: iff its
 *   value >= a threshold).  Neighbourhood: 4-connectivity
 *    or 8-connectivity (north_star), clipped at the image border.
 *   Output label of pixel p: 0 if background, else 1 + the minimum raster index
 *   of p's component (the unique canonical form; reading R3).
 *
 * Conventions shared by every entry point
 *   - Layout: contiguous row-major, row stride W, no pitch.  Batched: image b
 *     starts at byte offset b*H*W of `images`; its labels at element offset
 *     b*H*W of `labels_out`.  Labels are per image.
 *   - Memory: every pointer named d_* / images / labels_out / workspace is a
 *     CUDA device pointer on the current device; h_* pointers are host memory
 *     (page-locked for full copy bandwidth).  The CALLER owns all memory; the
 *     library keeps no state besides cached device attributes.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  *_async calls only enqueue work; they return before the
 *     GPU finishes.  Device faults surface at the caller's next synchronisation.
 *   - Errors: argument errors are detected on the host BEFORE anything is
 *     enqueued and reported as a status code; nothing is written.  A failed
 *     launch returns CCL_ERR_CUDA and ccl_last_cuda_error() gives the
 *     cudaError_t.  No exceptions or aborts cross the ABI.
 *   - Sizes: H >= 1, W >= 1, B >= 0 (B == 0 is a no-op returning CCL_OK);
 *     H*W must be <= 2^31-1 (labels are int32), else CCL_ERR_TOO_LARGE.
 *   - Determinism: output is bit-identical across runs, streams, tile
 *     configurations and GPU counts (the canonical form is unique).
 *   - Thread safety: reentrant; distinct streams may run concurrently.
 */
#ifndef CCL_B200_H
#define CCL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CCL_OK = 0,
    CCL_ERR_NULL = 1,          /* a required pointer is NULL                         */
    CCL_ERR_DIMS = 2,          /* H < 1, W < 1, B < 0, or bad strip geometry         */
    CCL_ERR_TOO_LARGE = 3,     /* H*W > 2^31-1 (labels would overflow int32)         */
    CCL_ERR_CONNECTIVITY = 4,  /* connectivity not in {4, 8}                         */
    CCL_ERR_ALIAS = 5,         /* input and output / workspace byte ranges overlap   */
    CCL_ERR_WORKSPACE = 6,     /* workspace smaller than ccl_workspace_bytes()       */
    CCL_ERR_CUDA = 7,          /* a CUDA runtime call or launch failed               */
    CCL_ERR_CONFIG = 8         /* unsupported tile configuration / threshold         */
} ccl_status_t;

/* Human-readable text for a status code (static storage, never NULL). */
const char* ccl_status_string(ccl_status_t status);

/* cudaError_t of the most recent CCL_ERR_CUDA returned on the calling thread. */
int ccl_last_cuda_error(void);

/* Device workspace (bytes) needed by the *_async entry points for B images of
 * H x W (3.7 bytes per pixel for 8192 x 8192): the
 * bit-packed foreground mask (1/8 B/px, rows padded to 32 px), per-run records
 * (4 B per run, sized for the worst case of alternating pixels: 2 B/px),
 * per-tile edge briefs (136 ints per 8-row tile), the boundary analysis'
 * union-find over edge slots (8 bytes per slot, one slot per edge-touching
 * local root; per tile enough for the worst case of the tile configuration
 * that needs the most -- 1.5 B/px), the K1 -> K2 ready flags and the lists of
 * run-dense tiles.  Sized for every tile configuration.  The strip stages
 * need more (ccl_strip_workspace_bytes).  Returns 0 for invalid arguments. */
size_t ccl_workspace_bytes(int64_t B, int64_t H, int64_t W, int connectivity);

/* Label one H x W image (device pointers).  Allocates its workspace stream-
 * ordered (cudaMallocAsync) on the legacy default stream and frees it there;
 * asynchronous to the host like every other launch on that stream. */
ccl_status_t ccl_label(const uint8_t* image, int64_t H, int64_t W, int connectivity,
                       int32_t* labels_out);

/* Label B independent H x W images (device pointers), labels per image.  Same
 * workspace policy as ccl_label. */
ccl_status_t ccl_label_batched(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                               int connectivity, int32_t* labels_out);

/* The hot path: the paper's three kernels enqueued on `stream`
 *   K1 local merge with coarse labeling   (Alg. 1; §2.1)
 *   K2 boundary analysis                  (Alg. 2; §2.2)
 *   K3 final link                         (§2.3)
 * using the caller's workspace (>= ccl_workspace_bytes(B,H,W,connectivity)
 * bytes, 256-byte aligned, contents need not be initialised).  `images` must
 * not overlap `labels_out` or `workspace`. */
ccl_status_t ccl_label_batched_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                     int connectivity, int32_t* labels_out,
                                     void* workspace, size_t workspace_bytes, void* stream);

/* As ccl_label_batched_async with an explicit tile height (rows per K1 thread
 * block: 8, 16 or 32; 0 = library default: the tallest of 32, 16, 8 whose
 * tiles number at least 4 per SM of the current device -- 32 for C3 / C4 /
 * C5-sized work, 8 for small images; CCL_TILE_AUTO=0 in the environment pins
 * the default to 16).  The tile width is fixed at 1024
 * pixels (32 lanes x 32 px).  Output is identical for every tile config
 * ("config independence"); unsupported values -> CCL_ERR_CONFIG. */
ccl_status_t ccl_label_batched_cfg_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                         int connectivity, int32_t* labels_out,
                                         void* workspace, size_t workspace_bytes,
                                         int tile_rows, void* stream);

/* As ccl_label_batched_cfg_async on grey-level images, with the binarisation
 * fused into K1's load ("binarize": output 255 if input >=
 * threshold; the paper thresholds its grey test images):
 * a pixel is foreground iff its value >= threshold.  threshold = 1 is the
 * default "nonzero" test; 0 makes every pixel foreground.  The labels are
 * those of ccl_label on the binarised image.  threshold outside 0..255 ->
 * CCL_ERR_CONFIG (nothing launched); other errors as above. */
ccl_status_t ccl_label_threshold_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                       int connectivity, int threshold, int32_t* labels_out,
                                       void* workspace, size_t workspace_bytes, int tile_rows,
                                       void* stream);

/* The three stages individually (same arguments as ccl_label_batched_cfg_async),
 * for per-kernel timing and stage tests.  They must be enqueued in this order on
 * one stream with the same workspace:
 *   ccl_stage_local_merge  K1: reads images; writes the bit-packed mask, the
 *                          per-run records, the edge briefs and the initial
 *                          edge-slot entries (workspace).
 *   ccl_stage_boundary     K2: unions every foreground edge that crosses a tile
 *                          boundary into the edge-slot union-find (workspace only).
 *   ccl_stage_link         K3: resolves the tile-edge roots to their final
 *                          labels (the last step of the boundary analysis,
 *                          done by K3's helper warps) and writes labels_out
 *                          for every pixel.                                */
ccl_status_t ccl_stage_local_merge(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                   int connectivity, void* workspace, size_t workspace_bytes,
                                   int tile_rows, void* stream);
ccl_status_t ccl_stage_boundary(int64_t B, int64_t H, int64_t W, int connectivity,
                                void* workspace, size_t workspace_bytes, int tile_rows,
                                void* stream);
ccl_status_t ccl_stage_link(int64_t B, int64_t H, int64_t W, int connectivity,
                            int32_t* labels_out, void* workspace, size_t workspace_bytes,
                            int tile_rows, void* stream);

/* The paper's comparison methods (Table 2; SURVEY.md 8(f)
 * NEXT-1), on B200, for measuring the paper's relative claims -- not product
 * paths.  Same problem, conventions and canonical output as ccl_label:
 *   CCL_METHOD_OPTIMIZED  this library's three-kernel path (= ccl_label_batched_async)
 *   CCL_METHOD_UF         conventional parallel UF [oliveira2010study]
 *                         (PAPER.md:37, 68-70): per-pixel local UF in shared
 *                         memory over {32,16,1} blocks, global merge of every
 *                         tile-boundary pixel, per-pixel link
 *   CCL_METHOD_LINE_UF    line-based UF [yonehara2015line]:
 *                         {512,1,1} row segments, global UF over all cells
 *   CCL_METHOD_LE         label equivalence: multi-pass;
 *                         reads a convergence flag back every iteration, so
 *                         this call SYNCHRONISES the stream and returns when done
 * Workspace: >= ccl_method_workspace_bytes(...) device bytes (0 = invalid
 * geometry or method).  Unknown method -> CCL_ERR_CONFIG; B or H > 65535 ->
 * CCL_ERR_DIMS (grid limits of the pixel-level launches). */
enum { CCL_METHOD_OPTIMIZED = 0, CCL_METHOD_UF = 1, CCL_METHOD_LINE_UF = 2, CCL_METHOD_LE = 3 };
size_t ccl_method_workspace_bytes(int64_t B, int64_t H, int64_t W, int connectivity, int method);
ccl_status_t ccl_label_method_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                    int connectivity, int method, int32_t* labels_out,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Equal-value mode: the paper's kernels compare raw
 * pixel values (dBuff[tid] == dBuff[tid-1], PAPER.md:104, 110, 123, 127, 294,
 * 299), so they label every region of equal value, background included, and
 * accept grey-level input; the SPEC CPU program adopts that.
 * Here: every pixel p gets the 0-BASED minimum raster index of its component
 * of equal-valued, 4- or 8-connected pixels -- no
 * background value, no +1.  Computed with the conventional-UF kernels
 * (ccl_label_method_async's CCL_METHOD_UF) under an equality predicate.
 * Workspace >= ccl_method_workspace_bytes(B, H, W, connectivity,
 * CCL_METHOD_UF).  Errors as ccl_label_method_async. */
ccl_status_t ccl_label_equal_async(const uint8_t* images, int64_t B, int64_t H, int64_t W,
                                   int connectivity, int32_t* labels_out, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* 3D volumes ("2D/3D grid"): B volumes of
 * D x H x W uint8 voxels, row-major (x fastest, then y, then z; volume b at
 * b*D*H*W), raster index (z*H + y)*W + x.  Foreground = nonzero; connectivity
 * 6 (faces) or 26 (faces, edges, corners), clipped.  labels_out: int32, 0 or
 * 1 + the minimum raster index of the voxel's component (per volume).  The
 * three phases over 32x4x4 bricks at voxel granularity (csrc/ccl_3d.cuh).
 * Workspace >= ccl_workspace_bytes_3d(...) (0 = invalid arguments).  Errors:
 * CCL_ERR_DIMS (sizes < 1, or grid limits: B*ceil(D/4) or ceil(H/4) > 65535),
 * CCL_ERR_TOO_LARGE (D*H*W > 2^31-1), CCL_ERR_CONNECTIVITY (not 6/26), else
 * as ccl_label_batched_async. */
size_t ccl_workspace_bytes_3d(int64_t B, int64_t D, int64_t H, int64_t W, int connectivity);
ccl_status_t ccl_label_3d_async(const uint8_t* volumes, int64_t B, int64_t D, int64_t H, int64_t W,
                                int connectivity, int32_t* labels_out, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Per-component statistics of a label map produced by ccl_label* (SURVEY.md
 * 8(f) NEXT-3; "the size and location of each dot").  For image
 * b the components are listed in increasing label order (= raster order of
 * their minimum pixel), so record k of image b is component k+1 of the
 * compacted numbering 1..K_b (SPEC.md:336 renumbering):
 *   label   its label in labels (1 + minimum raster index)
 *   area    number of pixels
 *   x_min, y_min, x_max, y_max   inclusive bounding box
 *   sum_x, sum_y   coordinate sums (centroid = sum / area)
 * labels: device int32 [B][H][W], canonical (as ccl_label writes them -- any
 * other content gives meaningless but memory-safe output); 16-byte aligned
 * labels with H*W % 4 == 0 take 128-bit loads, other layouts scalar ones.  stats: device,
 * B * max_components records (image b at b * max_components).  counts:
 * device int32[B], K_b; when K_b > max_components only the first
 * max_components records are written.  Workspace >= ccl_stats_workspace_bytes.
 * Asynchronous on `stream`.  Errors as for ccl_label (max_components < 1 ->
 * CCL_ERR_DIMS; B > 65535 -> CCL_ERR_DIMS). */
typedef struct {
    int32_t label, area, x_min, y_min, x_max, y_max;
    int64_t sum_x, sum_y;
} ccl_component_t;
size_t ccl_stats_workspace_bytes(int64_t B, int64_t H, int64_t W);
ccl_status_t ccl_component_stats_async(const int32_t* labels, int64_t B, int64_t H, int64_t W,
                                       int64_t max_components, ccl_component_t* stats,
                                       int32_t* counts, void* workspace, size_t workspace_bytes,
                                       void* stream);
/* As ccl_component_stats_async, and (relabel_out != NULL) also the compacted
 * label map (SPEC.md:336 renumbering): relabel_out[p] = k for a pixel of the
 * k-th component in label order (1..K_b per image, the record index + 1),
 * 0 for background; device int32 [B][H][W], must not overlap the other
 * buffers (CCL_ERR_ALIAS). */
ccl_status_t ccl_component_stats_relabel_async(const int32_t* labels, int64_t B, int64_t H, int64_t W,
                                               int64_t max_components, ccl_component_t* stats,
                                               int32_t* counts, int32_t* relabel_out, void* workspace,
                                               size_t workspace_bytes, void* stream);

/* The tile height (8, 16 or 32) that tile_rows = 0 selects for this geometry
 * on the current device (the rule of ccl_label_batched_cfg_async; the SM
 * count is queried).  Host-only.  Returns -1 on invalid dimensions. */
int ccl_default_tile_rows(int64_t B, int64_t H, int64_t W);

/* Number of K2 boundary work items for the given geometry and tile height:
 * horizontal tile-edge segments (one warp each) and vertical tile-edge pixels
 * (one thread each).  Host-only bookkeeping (cf. Eq. (1)-(2), PAPER.md:326-334,
 * which counts boundary cells for the paper's {32,16} blocks).  Returns -1 on
 * invalid arguments. */
int64_t ccl_boundary_work_items(int64_t B, int64_t H, int64_t W, int tile_rows,
                                int64_t* horizontal_segments, int64_t* vertical_pixels);

/* End-to-end entry (host buffers): enqueues on `stream`, in order, the copy of
 * h_images (B*H*W bytes) to the device, the three kernels, and the copy of the
 * labels back into h_labels (B*H*W int32).  Within one call the copies and the
 * kernels are serialised on `stream` (the kernels need the whole image and
 * the labels are final only after K3); callers overlap consecutive calls by
 * alternating two streams and scratch buffers, so one call's label copy runs
 * during the next call's image copy and kernels (paper_1708_08180_b200.
 * HostPipeline, bench.py's e2e).  d_scratch is caller-owned device memory of
 * >= ccl_host_scratch_bytes() bytes.  Returns after enqueueing; the caller
 * synchronises `stream` before reading h_labels.  h_images/h_labels should be
 * page-locked (cudaHostAlloc / cudaHostRegister) for asynchronous copies. */
size_t ccl_host_scratch_bytes(int64_t B, int64_t H, int64_t W, int connectivity);
ccl_status_t ccl_label_host_async(const uint8_t* h_images, int64_t B, int64_t H, int64_t W,
                                  int connectivity, int32_t* h_labels,
                                  void* d_scratch, size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Row-strip sharding of one image over k GPUs (north_star: "a single gigapixel
 * image splits into row strips whose edge-row labels are exchanged with NCCL
 * over NVLink, then merged by a cross-strip boundary-union and relabel pass").
 * Rank r owns rows [row0, row0 + rows) of an H_total x W image (strips are
 * contiguous and in rank order).  The result equals the unsharded labeling:
 * labels are 1 + GLOBAL raster indices (H_total * W must be <= 2^31 - 1).
 *
 *   ccl_strip_local    (rank r) K1 + K2 on the strip; writes the 4*W-int send
 *                      buffer: [0, W) labels of the strip's first row, [W, 2W)
 *                      of its last row (0 = background), [2W, 4W) for each of
 *                      those 2W slots the first slot with the same label
 *                      (-1: background).  The workspace carries state to
 *                      finalize (pass the same buffer, unchanged).
 *   caller             all-gather of the k send buffers into gathered
 *                      (k * 4 * W int32, rank order) -- e.g. ncclAllGather.
 *   ccl_strip_finalize (rank r) min-label union over the k*2W slots (same-label
 *                      slots of a strip; 4-/8-adjacent slots across every strip
 *                      cut); K3 writes labels_out, taking for each component on
 *                      a strip boundary the minimum label of its slot set.
 * Six launches per step: local = K1, K2, strip edges, strip reps; finalize =
 * slot union (a min-label union-find over the k*2W slots), K3.
 * Workspace: >= ccl_strip_workspace_bytes(rows, W, k, connectivity), the same
 * buffer for both calls (ccl_workspace_bytes of the strip plus 4 B per edge
 * slot for the strip marks and 16 B per boundary slot for the slot
 * union-find: about 4.5 B/px).  Errors as above; CCL_ERR_DIMS also for rank/k/row0
 * out of range. */
size_t ccl_strip_workspace_bytes(int64_t rows, int64_t W, int k, int connectivity);
ccl_status_t ccl_strip_local(const uint8_t* strip, int64_t rows, int64_t W, int64_t row0, int64_t H_total,
                             int connectivity, int k, int32_t* send, int32_t* labels_out,
                             void* workspace, size_t workspace_bytes, void* stream);
ccl_status_t ccl_strip_finalize(const int32_t* gathered, int k, int rank, int64_t rows, int64_t W,
                                int64_t row0, int64_t H_total, int connectivity, int32_t* labels_out,
                                void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CCL_B200_H */
