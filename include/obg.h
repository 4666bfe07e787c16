/*
 * obg.h -- C ABI of the B200 octree background-model hot path (libobg.so).
 *
 * Drop-in boundary for the octabg reference's build / prune / merge / classify
 * path (reference: /root/reference/pkg/src/octabg/).  Every entry point takes
 * plain device pointers and sizes plus a CUDA stream handle (`void*` holding a
 * cudaStream_t, NULL = legacy default stream).  Buffers are caller-allocated
 * and caller-owned; the library holds no persistent allocations and no global
 * mutable state other than a per-device launch-configuration cache, so calls
 * on different streams/threads are safe.
 *
 * Status: 0 = OK, negative = error (see OBG_E*).  obg_last_error() returns a
 * thread-local message for the last failing call on the calling thread.
 *
 * Data layout:
 *   frames   u8  [n_frames][height][width][3]  (HWC RGB, the reference's
 *                                               (h, w, 3) uint8 frames)
 *   pyramid  u32 [obg_pyramid_words(L)]        one octree = per-level presence
 *            bitsets, level 1..L concatenated (level l at
 *            obg_level_offset(L, l)); bit c of level l <=> the node whose
 *            path code (octree.py:70-80, l octal digits) is c exists.  Level-l
 *            word count = max(1, 8^l / 32).  The child mask byte of node p at
 *            level l (octree.py:217-227) is byte p of level l+1.
 *   cube     u32 [obg_cube_words(L)]           classify operand: leaf bitset in
 *            "RGB cube" order, idx = R'<<2L | G'<<L | B' with C' = C >> (8-L)
 *            (max(1, 8^L/32) words); for L = 7 followed by a 2-bit state per
 *            L=6 cell (16384 words: some / all of its 8 leaves present), 32
 *            words of cell counts and the L=6 bitset of full cells (8192
 *            words) -- what the L = 7 classify picks its kernel by.
 *   mask     u8  [n_frames][height][width]     0/1 (numpy bool layout), or
 *            bit-packed u8 [n_frames][ceil(h*w/8)], LSB-first per frame.
 */
#ifndef OBG_H
#define OBG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OBG_OK            0
#define OBG_EINVAL       -1   /* bad argument (maps to ValueError) */
#define OBG_EUNSUPPORTED -2   /* valid but unsupported configuration */
#define OBG_ECUDA        -3   /* CUDA runtime / launch failure */
#define OBG_EFORMAT      -4   /* malformed frame / mask file (maps to FormatError, with a byte offset) */
#define OBG_EIO          -5   /* file system error */

#define OBG_WS_ZEROED   1    /* obg_build_presence flag */

#define OBG_MASK_U8     0
#define OBG_MASK_PACKED 1
/* OR-ed into obg_classify's mask_format: the previous work on `stream` is the
 * obg_build_model that produced cube_bits.  The classify kernel is then
 * launched as a programmatic dependent of the merge kernel (its CTAs are
 * placed while the merge drains and wait for it on the device), which removes
 * the launch gap between the two.  Only valid right after obg_build_model on
 * the same stream; without the bit the launch is ordinary stream order.
 * Honoured when the environment sets OBG_PDL=2 (measured: -1.3 us on a
 * 146 us step, +2.4 us on a 392 us one, so it is off by default; the merge
 * kernel inside obg_build_model is always a dependent of the build kernel). */
#define OBG_MASK_AFTER_MODEL 0x100

/* ABI version of this header (bumped on incompatible change). */
int obg_abi_version(void);

/* Thread-local description of the last error on this thread ("" if none). */
const char* obg_last_error(void);

/* Sizes of the layouts above, in 32-bit words.  levels in 1..8, else -1. */
int64_t obg_pyramid_words(int levels);
int64_t obg_level_offset(int levels, int level);
int64_t obg_cube_words(int levels);

/* Scratch needed by obg_build_presence, in bytes. */
int64_t obg_build_workspace_bytes(int n_trees, int n_regions, int levels);

/* Path code per pixel, reference octree order.
 * Replaces pack_codes (octree.py:83-90): codes[i] = (SPREAD_R[r] | SPREAD_G[g]
 * | SPREAD_B[b]) >> 3*(8-levels) for pixel i = pixels[3i..3i+2]. */
int obg_pack_codes(const uint8_t* pixels, int64_t n_pixels, int levels,
                   uint32_t* codes, void* stream);

/* Per-(group, region) presence octrees of a batch of training frames.
 * Replaces the build loop of build_background_model (model.py:166-179) and
 * build_frame_tree (model.py:93-109): frames are split into
 * n_groups = n_frames / group_size consecutive groups (a trailing partial
 * group is dropped, model.py:166-167); each group and grid region
 * (region_bounds, model.py:69-75) yields one tree holding every quantized
 * colour its pixels carry.
 *   out_pyramids : u32 [n_groups][grid_rows*grid_cols][obg_pyramid_words(L)]
 *   out_counts   : optional (NULL = skip) u32 [n_groups][R*C][8^L], per-leaf
 *                  pixel occupancy histogram in path-code order (a superset of
 *                  the reference, which stores presence only; oracle is
 *                  np.bincount(pack_codes(block)))
 *   workspace    : >= obg_build_workspace_bytes(n_groups, R*C, L) bytes.  It is
 *                  returned all-zero; pass OBG_WS_ZEROED in flags when it is
 *                  all-zero on entry (e.g. a kept workspace) to skip clearing it. */
int obg_build_presence(const uint8_t* frames, int n_frames, int height, int width,
                       int levels, int grid_rows, int grid_cols, int group_size,
                       uint32_t* out_pyramids, uint32_t* out_counts,
                       void* workspace, int64_t workspace_bytes, int flags, void* stream);

/* build_background_model on the device in one call (model.py:157-185):
 * obg_build_presence + obg_merge with no memsets.  tree_pyramids is scratch
 * of obg_build_presence's out_pyramids size; out_merged u32 [R*C][PW];
 * out_cube u32 [R*C][obg_cube_words(L)] (the classify operand). */
int obg_build_model(const uint8_t* frames, int n_frames, int height, int width,
                    int levels, int grid_rows, int grid_cols, int group_size, int64_t k_min,
                    uint32_t* tree_pyramids, uint32_t* out_merged, uint32_t* out_cube,
                    void* workspace, int64_t workspace_bytes, int flags, void* stream);

/* Pyramids from leaf-level bitsets (path-code order, max(1,8^L/32) words per
 * tree): every interior level is the OR-reduction of the level below, i.e.
 * the nodes a tree built by Octree.store_code (octree.py:158-169) creates. */
int obg_pyramid_from_leaves(const uint32_t* leaves, int n_trees, int levels,
                            uint32_t* out_pyramids, void* stream);

/* Octree.prune (octree.py:193-204, _copy_truncated 284-290) on n_trees
 * pyramids: the result keeps levels 1..new_levels (dead-end nodes included). */
int obg_prune(const uint32_t* pyramids, int n_trees, int levels, int new_levels,
              uint32_t* out_pyramids, void* stream);

/* Per-node tree counts for merge_trees (model.py:112-154).
 * pyramids: u32 [n_trees][n_regions][PW]; counts: u32 [n_regions][PW*32],
 * counts[r][w*32+b] = number of input trees of region r holding node (w, b). */
int obg_merge_counts(const uint32_t* pyramids, int n_trees, int n_regions, int levels,
                     uint32_t* counts, void* stream);

/* counts >= k_min -> merged pyramids u32 [n_regions][PW].  The host computes
 * k_min = min{k >= 1 : k / total >= threshold} in IEEE double exactly as
 * model.py:152 compares. */
int obg_merge_threshold(const uint32_t* counts, int n_regions, int levels, int64_t k_min,
                        uint32_t* out_pyramids, uint32_t* out_cube, void* stream);

/* Fused obg_merge_counts + obg_merge_threshold (single GPU).  For both merge
 * entry points, out_cube (nullable) additionally receives the merged leaf
 * level in cube order, u32 [n_regions][obg_cube_words(L)] -- the classify
 * operand, as obg_leaf_cube would produce it. */
int obg_merge(const uint32_t* pyramids, int n_trees, int n_regions, int levels,
              int64_t k_min, uint32_t* out_pyramids, uint32_t* out_cube, void* stream);

/* Leaf level of n pyramids -> cube-order bitsets u32 [n][obg_cube_words(L)]
 * (the classify operand; detect.py:46 reads only full-depth leaves). */
int obg_leaf_cube(const uint32_t* pyramids, int n_trees, int levels,
                  uint32_t* cube, void* stream);

/* Foreground masks.  Replaces detect_octree (detect.py:22-53): pixel is
 * foreground iff its quantized colour is not a full-depth leaf of its
 * region's tree (empty tree => all foreground).
 *   cube_bits : u32 [grid_rows*grid_cols][obg_cube_words(L)] from obg_leaf_cube
 *   mask      : OBG_MASK_U8 -> u8 [n][h][w] 0/1; OBG_MASK_PACKED -> u8
 *               [n][ceil(h*w/8)], pixel i of a frame at bit i%8 of byte i/8. */
int obg_classify(const uint8_t* frames, int n_frames, int height, int width, int levels,
                 int grid_rows, int grid_cols, const uint32_t* cube_bits,
                 uint8_t* mask, int mask_format, void* stream);

/* Classification fused with evaluation: the confusion counts of the
 * predicted foreground against a ground-truth mask, no mask written.
 * Replaces detect_octree followed by evaluation.accumulate
 * (evaluation.py:38-53; foreground is the positive class).
 *   truth  : same layout as obg_classify's mask (truth_format OBG_MASK_U8:
 *            any nonzero byte = foreground, e.g. 0/1 or 0/255 PGM values;
 *            OBG_MASK_PACKED: bit-packed).
 *   counts : device u64 [4] = tn, tp, fn, fp, ADDED to (like accumulate's
 *            stats argument). */
int obg_classify_confusion(const uint8_t* frames, int n_frames, int height, int width, int levels,
                           int grid_rows, int grid_cols, const uint32_t* cube_bits,
                           const uint8_t* truth, int truth_format, uint64_t* counts, void* stream);

/* detect_octree with the reference's own signature (detect.py:22-53: one
 * numpy frame in, one numpy bool mask out; the reference CLI calls it per
 * frame, cli.py:181-187): HOST frames u8 [n][h][w][3] in, HOST masks u8
 * [n][h][w] 0/1 out, cube_bits on the device as for obg_classify.  Frames
 * are staged through pinned memory by the host copy pool and moved with
 * asynchronous copies pipelined in halves around the classify kernel; the
 * call returns when the masks are in `mask`.  Staging buffers are cached per
 * calling thread (obg_host_stage_release frees the caller's). */
int obg_detect_host(const uint8_t* frames, int n_frames, int height, int width, int levels,
                    int grid_rows, int grid_cols, const uint32_t* cube_bits, uint8_t* mask,
                    void* stream);
void obg_host_stage_release(void);

/* Preorder child-mask serialization of one pyramid (Octree.to_bytes,
 * octree.py:217-227, 258-267) computed on the device.
 *   has_root : 1 if the tree has a root node.
 *   out      : device buffer of >= 1 + popcount(pyramid) bytes.
 *   n_out    : host pointer receiving the byte count (synchronises stream).
 *   workspace: >= obg_serialize_workspace_bytes(L) bytes. */
int64_t obg_serialize_workspace_bytes(int levels);
int obg_serialize(const uint32_t* pyramid, int levels, int has_root, uint8_t* out,
                  int64_t out_capacity, int64_t* n_out, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* ---- frame ingest (host only; frame_io.py) -------------------------------
 * Binary PPM (P6, kind 6) frames / PGM (P5, kind 5) masks with the
 * reference's header rules, messages and byte offsets (frame_io.py:22-104).
 *
 * Header + payload-size check of an in-memory file.  On OBG_EFORMAT,
 * *err_offset is the reference's FormatError offset. */
int obg_pnm_header(const uint8_t* data, int64_t size, int kind, int64_t* width,
                   int64_t* height, int64_t* payload, int64_t* err_offset);

/* Read n same-sized files (FrameSequence.load_all, frame_io.py:157-176)
 * straight into `out` (n x height x width x (3 | 1) bytes, e.g. pinned host
 * memory for the overlapped H2D pipeline) with n_threads host threads
 * (<= 0: all cores).  On error *bad_index is the first failing file. */
int obg_read_pnm_files(const char* const* paths, int n_files, int kind, int64_t width,
                       int64_t height, uint8_t* out, int n_threads, int* bad_index,
                       int64_t* err_offset);

/* Write n masks (u8, nonzero = foreground) as P5 PGM files of 0/255
 * (write_mask_pgm / save_mask, frame_io.py:107-125). */
int obg_write_pgm_masks(const uint8_t* masks, int n_masks, int64_t width, int64_t height,
                        const char* const* paths, int n_threads);

/* Copy n host blocks of bytes_each bytes, srcs[i] -> dst + i * bytes_each
 * (e.g. a list of frames into one pinned staging buffer), split into 256 KiB
 * pieces over a persistent pool of host threads, with non-temporal stores
 * (see obg_host_copy).  Host only. */
int obg_host_gather(const uint8_t* const* srcs, int n, int64_t bytes_each, uint8_t* dst);

/* One host block copied by the same pool.  streaming != 0: non-temporal
 * stores, for a pinned destination the GPU reads next (ordinary stores leave
 * the lines dirty in the pool cores' caches and the DMA snoops them out:
 * ~12 GB/s instead of ~50 for a 6 MB frame); 0: ordinary stores, for data
 * the host reads next.  obg_host_gather always streams.  Host only. */
int obg_host_copy(const uint8_t* src, int64_t bytes, uint8_t* dst, int streaming);

/* Parse one non-empty preorder child-mask tree (Octree.from_bytes /
 * decode_tree, octree.py:229-237, 250-281) at data[pos..n) into a host
 * path-order pyramid (u32 [obg_pyramid_words(depth)]).  On OBG_EFORMAT,
 * *err_kind is 0 ("truncated octree data") or 1 ("octree node below leaf
 * depth") and *err_offset the reference's byte offset; *end_pos is the byte
 * after the tree.  Host only. */
int obg_decode_tree(const uint8_t* data, int64_t n, int64_t pos, int depth, uint32_t* pyramid,
                    int64_t* end_pos, int64_t* err_offset, int* err_kind);

/* The same parse emitting the nodes below the root in preorder as
 * codes[k] (path code) / levels[k] (1..depth), *n_nodes of them -- O(nodes)
 * for sparse trees; each level's codes come out ascending.  capacity >=
 * n - pos - 1 always suffices.  Errors as obg_decode_tree.  Host only. */
int obg_decode_tree_codes(const uint8_t* data, int64_t n, int64_t pos, int depth, uint32_t* codes,
                          uint8_t* levels, int64_t capacity, int64_t* n_nodes, int64_t* end_pos,
                          int64_t* err_offset, int* err_kind);

/* ---- sharded model build (distributed.py) -----------------
 * Per-node tree counts of this rank's frames: the build of obg_build_model
 * without its threshold.  counts: device u32 [R*C][pyramid_words][32], word w
 * in the cube-order level layout (level_offset(l) + cube word), bit b at
 * [w][b] -- sum them over ranks (all-reduce), then obg_threshold_counts with
 * k_min from the global tree total gives every rank the merged model
 * (out_merged path-order pyramids [R*C][PW], out_cube classify operands
 * [R*C][obg_cube_words]). */
int obg_build_counts(const uint8_t* frames, int n_frames, int height, int width, int levels,
                     int grid_rows, int grid_cols, int group_size, uint32_t* counts,
                     void* workspace, int64_t workspace_bytes, int flags, void* stream);
int obg_threshold_counts(const uint32_t* counts, int n_regions, int levels, int64_t k_min,
                         uint32_t* out_merged, uint32_t* out_cube, void* stream);

/* ---- comparison baselines (detect.py:56-83) -------------------------------
 * Frame difference (detect_frame_diff, detect.py:56-63): mask i (u8 0/1,
 * [n_pairs][pixels]) is 1 where some channel of cur[i] differs from prev[i]
 * by strictly more than diff_threshold.  prev / cur are u8 [n_pairs][pixels][3];
 * cur == prev + 3 * pixels (consecutive frames of one buffer) reads every
 * frame once. */
int obg_frame_diff(const uint8_t* prev, const uint8_t* cur, int n_pairs, int64_t pixels,
                   int diff_threshold, uint8_t* masks, void* stream);

/* Running mean (detect_running_average, detect.py:66-83) over n_frames
 * consecutive frames: for t = 0..n-1, mask t = max_c |x_c - avg_c| >
 * diff_threshold with the mean before the update, then
 * avg += (x - avg) / (frames_seen + t + 1) in IEEE binary64 (bit-identical
 * to the reference's numpy).  average: device f64 [pixels][3], updated in
 * place; masks: u8 0/1 [n_frames][pixels]. */
int obg_running_average(const uint8_t* frames, int n_frames, int64_t pixels, int64_t frames_seen,
                        double* average, int diff_threshold, uint8_t* masks, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OBG_H */
