/*
 * mergepath_b200.h -- C ABI of the B200-native Merge Path library
 * (libmergepath_b200.so, built from paper_1406_2628_b200/csrc/).
 *
 * This is the drop-in boundary.  The reference exposes its hot path as C++
 * templates over <T, Comp> (no compiled ABI at all):
 *   diagonal_search / partition          core.hpp:120-146
 *   sequential_merge                     core.hpp:148-180
 *   parallel_merge[_into]                parallel.hpp:151-179
 *   segmented_parallel_merge[_into]      parallel.hpp:200-236
 *   plan_segments                        parallel.hpp:258-292
 *   parallel_merge_checksum / segmented_parallel_merge_checksum
 *                                        parallel.hpp:181-198, :238-256
 *   parallel_merge_sort                  sort.hpp:132-148
 *   cache_efficient_parallel_sort        sort.hpp:150-195
 * The drop-in C++ headers in include/mergepath/ keep those exact template
 * signatures and forward every supported (T, Comp) pair to the entry points
 * below; INTEGRATION.md shows the binding.  Plain pointers and sizes only.
 *
 * Conventions
 *   - Device entry points (no suffix) take DEVICE pointers and a
 *     cudaStream_t passed as void*; they are asynchronous on that stream.
 *   - *_host entry points take HOST pointers (pageable or pinned), stage
 *     through the GPU `device` and return when the result is in host memory.
 *   - Every call returns an mp_status; mp_last_error() describes the last
 *     failure on the calling thread.
 *   - Ties: equal keys take A first (core.hpp:79-87), so merges are stable
 *     with A as the left operand and sorts are stable w.r.t. input index.
 *   - Optional uint32 values travel with their keys (SoA records ordered by
 *     key only).  Pass NULL for keys-only.  MP_KEY_ELEMENT keys carry their
 *     own tag and take no separate values.
 */
#ifndef MERGEPATH_B200_H
#define MERGEPATH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mp_key_type {
  MP_KEY_U32 = 0,     /* std::less<uint32_t> */
  MP_KEY_I32 = 1,     /* std::less<int32_t> */
  MP_KEY_F32 = 2,     /* IEEE 754 totalOrder on float32 (-0.0 < +0.0) */
  MP_KEY_U64 = 3,     /* std::less<uint64_t> */
  MP_KEY_I64 = 4,     /* std::less<int64_t> */
  MP_KEY_ELEMENT = 5  /* reference `element` {int64 key; uint32 tag}, 16 B,
                         ordered by key only (core.hpp:39-53) */
} mp_key_type;

typedef enum mp_status {
  MP_OK = 0,
  MP_ERR_INVALID = 1,     /* std::invalid_argument in the reference */
  MP_ERR_CUDA = 2,        /* CUDA launch / runtime failure */
  MP_ERR_OOM = 3,         /* device or pinned allocation failed */
  MP_ERR_UNSUPPORTED = 4, /* key type / value combination not supported */
  MP_ERR_IO = 5           /* file I/O failure or truncated key file
                             (std::runtime_error in dataio.cpp) */
} mp_status;

/* Message for the last non-OK status on this thread ("" if none). */
const char *mp_last_error(void);
/* ABI version (major*100 + minor). */
int mp_abi_version(void);
/* Kernels this library has launched in the process so far (all threads). */
uint64_t mp_launch_count(void);
/* Size in bytes of one key of `key_type` (0 if unknown). */
uint64_t mp_key_size(int key_type);

/* ---- partition (core.hpp:120-146) ------------------------------------- */
/* a_offs[i] = a_off of the merge path on diagonal floor(i*(na+nb)/p),
 * i = 0..p (p+1 device uint64 entries); b_off = diagonal - a_off.
 * p == 0 -> MP_ERR_INVALID (core.hpp:139-140).  `comparisons` (device
 * uint64, may be NULL) accumulates the element comparisons of the p+1
 * searches exactly as the reference counts them (core.hpp:120-132). */
int mp_partition(int key_type, const void *a, uint64_t na, const void *b,
                 uint64_t nb, uint64_t p, uint64_t *a_offs,
                 uint64_t *comparisons, void *stream);

/* a_offs[k] = a_off on diagonal diags[k] (clamped to na+nb), k < count.
 * `comparisons` as for mp_partition. */
int mp_diagonal_search(int key_type, const void *a, uint64_t na,
                       const void *b, uint64_t nb, const uint64_t *diags,
                       uint64_t count, uint64_t *a_offs,
                       uint64_t *comparisons, void *stream);

/* ---- merge (parallel.hpp:151-179, :200-236) --------------------------- */
/* out[0, na+nb) = stable merge of A and B.  Values optional (all three of
 * a_vals/b_vals/out_vals, or none).  Output must not overlap the inputs. */
int mp_merge(int key_type, const void *a, const uint32_t *a_vals, uint64_t na,
             const void *b, const uint32_t *b_vals, uint64_t nb, void *out,
             uint32_t *out_vals, void *stream);

/* The same merge in two stream-ordered phases over a caller-owned device
 * workspace (for CUDA graphs, overlap and per-kernel timing):
 *   mp_merge_plan    -- K1: tile split points into `workspace`
 *   mp_merge_execute -- K2: the tile merge reading those split points
 * mp_merge == plan + execute.  The workspace depends only on the key type
 * and na + nb. */
uint64_t mp_merge_workspace_bytes(int key_type, uint64_t na, uint64_t nb);
int mp_merge_plan(int key_type, const void *a, uint64_t na, const void *b,
                  uint64_t nb, void *workspace, void *stream);
int mp_merge_execute(int key_type, const void *a, const uint32_t *a_vals,
                     uint64_t na, const void *b, const uint32_t *b_vals,
                     uint64_t nb, void *out, uint32_t *out_vals,
                     const void *workspace, void *stream);

/* Register-sink merge (parallel.hpp:181-198): *sum (device uint64) =
 * sum over merged positions i of (i+1)*mix64(key_i) (core.hpp:200-245),
 * without writing the merged array.  Integer key types and ELEMENT;
 * F32 keys are bit-cast. */
int mp_merge_checksum(int key_type, const void *a, uint64_t na, const void *b,
                      uint64_t nb, uint64_t *sum, void *stream);

/* ---- sort (sort.hpp:132-195) ------------------------------------------ */
/* Stable sort of keys[0,n) in place (vals optional, permuted alongside).
 * scratch may be NULL (stream-ordered pool allocation) or a device buffer of
 * at least mp_sort_scratch_bytes() bytes. */
uint64_t mp_sort_scratch_bytes(int key_type, int with_vals, uint64_t n);
int mp_sort(int key_type, void *keys, uint32_t *vals, uint64_t n,
            void *scratch, uint64_t scratch_bytes, void *stream);
/* Out-of-place: sorted keys_in (+ vals_in) land in keys_out (+ vals_out);
 * the inputs are not modified (the block sort reads them directly, saving
 * the copy parallel_merge_sort makes, sort.hpp:137).  May alias (== mp_sort). */
int mp_sort_to(int key_type, const void *keys_in, const uint32_t *vals_in,
               void *keys_out, uint32_t *vals_out, uint64_t n, void *scratch,
               uint64_t scratch_bytes, void *stream);

/* ---- segmented-merge schedule (parallel.hpp:90-145, :258-292) --------- */
/* Windows of L = cache_elems/3 outputs; ceil((na+nb)/L) of them.
 * start_a[k] (device) = a_off where window k starts (diagonal k*L).
 * plan_comparisons / merge_comparisons (device uint64, may be NULL)
 * accumulate the reference's counters: plan_segments' end-of-window
 * searches and the p_eff window-local worker searches of
 * segmented_parallel_merge.  p == 0 or cache_elems < 3 -> MP_ERR_INVALID. */
uint64_t mp_segment_iterations(uint64_t na, uint64_t nb, uint64_t cache_elems);
int mp_segment_plan(int key_type, const void *a, uint64_t na, const void *b,
                    uint64_t nb, uint64_t p, uint64_t cache_elems,
                    uint64_t *start_a, uint64_t *plan_comparisons,
                    uint64_t *merge_comparisons, void *stream);

/* ---- host-buffer entry points (synchronous) --------------------------- */
/* Counters (`comparisons`, `*_comparisons`) are host uint64 here, may be
 * NULL, and accumulate (+=) like the reference's stats pointers.
 * mp_merge_host / mp_sort_host stream chunks over PCIe (H2D, kernels, D2H
 * overlapped on three streams).  Page-locked buffers are DMA'd directly;
 * pageable ones (a plain std::vector) are staged chunk by chunk through
 * pinned slots by a pool of host threads, overlapped with the transfers. */
int mp_partition_host(int key_type, const void *a, uint64_t na, const void *b,
                      uint64_t nb, uint64_t p, uint64_t *a_offs,
                      uint64_t *comparisons, int device);
int mp_diagonal_search_host(int key_type, const void *a, uint64_t na,
                            const void *b, uint64_t nb, const uint64_t *diags,
                            uint64_t count, uint64_t *a_offs,
                            uint64_t *comparisons, int device);
int mp_segment_plan_host(int key_type, const void *a, uint64_t na,
                         const void *b, uint64_t nb, uint64_t p,
                         uint64_t cache_elems, uint64_t *start_a,
                         uint64_t *start_b, uint64_t *plan_comparisons,
                         uint64_t *merge_comparisons, int device);
int mp_merge_host(int key_type, const void *a, const uint32_t *a_vals,
                  uint64_t na, const void *b, const uint32_t *b_vals,
                  uint64_t nb, void *out, uint32_t *out_vals, int device);
int mp_sort_host(int key_type, const void *keys, const uint32_t *vals,
                 uint64_t n, void *out_keys, uint32_t *out_vals, int device);
int mp_merge_checksum_host(int key_type, const void *a, uint64_t na,
                           const void *b, uint64_t nb, uint64_t *sum,
                           int device);

/* ---- multi-GPU: merging sharded sequences over NVLink ----------------- */
/* One contiguous piece (shard) of a sorted sequence; keys (and optional
 * values) are device pointers, possibly peer-mapped memory of another GPU
 * (mp_ipc_import). */
typedef struct mp_piece {
  const void *keys;
  const uint32_t *vals;
  uint64_t len;
} mp_piece;

/* out[0, out_end - out_begin) = positions [out_begin, out_end) of the stable
 * merge of A = a[0] ++ a[1] ++ ... and B = b[0] ++ ... (1..16 pieces each).
 * Asynchronous on `stream` (no host synchronisation): the tile split points
 * of the range are searched over the virtual index spaces on the device,
 * then each tile's windows are read straight from the piece pointers --
 * remote pieces over NVLink inside the tile loads (no staging copy).  The
 * caller orders the pieces' producers before `stream` (events / mp_signal).
 * out_vals non-NULL => every non-empty piece must carry vals. */
int mp_merge_pieces(int key_type, const mp_piece *a, int na_pieces,
                    const mp_piece *b, int nb_pieces, uint64_t out_begin,
                    uint64_t out_end, void *out, uint32_t *out_vals,
                    void *stream);

/* ---- multi-GPU in one process: shard tables --------------------------- */
/* A shard of a sequence on one GPU (keys, optional values: device pointers
 * on `device`). */
typedef struct mp_shard {
  int device;
  void *keys;
  uint32_t *vals;
  uint64_t len;
} mp_shard;

/* Stable merge of A = a[0] ++ ... ++ a[na-1] and B = b[0] ++ ... (each 1..16
 * shards, any devices) into the output shards: out[g] receives merged
 * positions [len(out[0..g)), + out[g].len) and is computed ON out[g].device,
 * its windows read straight from the input shards' devices (peer access is
 * enabled; NVLink pull inside the tile loads).  sum(out.len) must equal
 * |A| + |B| (parallel.hpp:155-156).  Values ride along when any output
 * shard has a vals pointer (then every non-empty shard carries them).
 * streams == NULL: blocking (all involved devices synchronised at entry,
 * the call returns when the output is complete).  Otherwise streams[g] (on
 * out[g].device) for each output shard: asynchronous, ordered after all
 * prior work on every given stream and before all later work on any of
 * them (cross-device events), so inputs may be produced on those streams. */
int mp_multi_merge(int key_type, const mp_shard *a, int na, const mp_shard *b, int nb,
                   const mp_shard *out, int nout, void *const *streams);
/* In-place stable sort of X = x[0] ++ ... ++ x[P-1] (P = 1..16 shards, any
 * devices; values ride along when any shard has a vals pointer): afterwards x[g]
 * holds sorted positions [len(x[0..g)), + x[g].len).  Each shard is sorted
 * on its device (mp_sort), then ceil(log2 P) rounds merge rank groups
 * (left group = A: stable w.r.t. the input order) with every shard keeping
 * its length; one scratch buffer per shard from the library pool.
 * `streams` as for mp_multi_merge (one per shard). */
int mp_multi_sort(int key_type, const mp_shard *x, int P, void *const *streams);

/* a_offs[k] = a_off of the merge path of the piece lists on diagonal
 * diags[k] (clamped to |A| + |B|): the multi-GPU analogue of
 * mp_diagonal_search (diags and a_offs are device arrays).  Used to place a
 * caller's own output slices and to count the NVLink traffic of a merge. */
int mp_pieces_partition(int key_type, const mp_piece *a, int na_pieces,
                        const mp_piece *b, int nb_pieces, const uint64_t *diags,
                        uint64_t count, uint64_t *a_offs, void *stream);
/* Copy `bytes` (16-byte aligned pointers, size a multiple of 16) with SM
 * vector loads -- the merge kernels' peer-window access pattern; with a
 * peer-mapped `src` it measures the NVLink pull rate (tools/nvlink_probe.py,
 * bench.py --gpus N). */
int mp_peer_copy(void *dst, const void *src, uint64_t bytes, void *stream);

/* CUDA IPC for shards owned by other processes: export writes a 64-byte
 * handle of the allocation holding dev_ptr plus dev_ptr's offset in it;
 * import maps it (once per allocation, peer access enabled lazily) and
 * returns the mapped address of the same byte. */
int mp_ipc_export(const void *dev_ptr, void *handle64, uint64_t *offset);
int mp_ipc_import(const void *handle64, uint64_t offset, void **dev_ptr);
/* Mappings are cached per (importing device, allocation) and reference
 * counted: each import takes a reference, mp_ipc_close(ptr) (any pointer an
 * import returned) drops one and unmaps the allocation at zero.
 * mp_ipc_open_count() = allocations currently mapped by this process. */
int mp_ipc_close(const void *dev_ptr);
uint64_t mp_ipc_open_count(void);

/* Stream-ordered flags for ordering work across processes and GPUs without
 * host synchronisation: mp_signal writes `value` to the 8-byte device word
 * `flag` (local or peer-mapped) after all prior work of `stream`, with a
 * system-scope fence; mp_wait makes `stream` wait until *flag >= value (the
 * stream's front end polls; no SM spins).  Use monotonically growing
 * generation numbers. */
int mp_signal(uint64_t *flag, uint64_t value, void *stream);
int mp_wait(const uint64_t *flag, uint64_t value, void *stream);

/* ---- memory ------------------------------------------------------------ */
/* Scratch comes from a library-private stream-ordered pool per device that
 * keeps its memory between calls; mp_release(device) waits for the device,
 * frees the host-pipeline slot buffers (device slots and the pinned staging
 * slots of pageable host calls) and trims that pool to zero. */
int mp_release(int device);
/* Page-locked host memory (cudaHostAlloc, portable across devices): host
 * buffers the DMA engines read directly.  NULL on failure. */
void *mp_host_alloc(uint64_t bytes);
int mp_host_free(void *p);

/* ---- synthetic inputs (bench/tests; SURVEY.md §8d generator) ---------- */
/* out[k] = config key kind `gen_kind` at global index first+k for `seed`:
 * 0 u32 = x>>32; 1 i32 in [0,1024) = x>>54; 2 u64 = x; 3 u64 < 2^40;
 * 4 u64 in [2^40, 2^64); 5 f32 Normal(0,1) (Box-Muller, cosine branch, in
 * double); 6 f32 Exp(1).  x_i = mix64(seed + i*0x9E3779B97F4A7C15).
 * Kinds 5/6 use the device's double-precision log/cospi: bytes can differ in
 * the last float ulp from a host-libm generator, so parity checks always run
 * on copies of the same device-generated bytes. */
int mp_generate(int gen_kind, uint64_t seed, uint64_t first, uint64_t n,
                void *out, void *stream);

/* ---- key files (dataio.hpp:5-25, dataio.cpp:33-98) -------------------- */
/* Binary: "MPKB0001", u64 LE count, count x i64 LE keys.  Text: one integer
 * per line (blank lines skipped).  Readers detect the format from the magic.
 * Unparsable text -> MP_ERR_INVALID (naming the line); open/read/write
 * failure or a truncated binary file -> MP_ERR_IO. */
int mp_keyfile_count(const char *path, uint64_t *count, int *is_binary);
int mp_keyfile_read(const char *path, int64_t *keys, uint64_t capacity,
                    uint64_t *count);
int mp_keyfile_write(const char *path, const int64_t *keys, uint64_t count,
                     int binary);
/* File -> device memory (i64 keys, MP_KEY_I64): a binary file is streamed
 * through two pinned 32 MiB buffers, pread of chunk k+1 overlapping the H2D
 * copy of chunk k.  Synchronous w.r.t. `stream` on return. */
int mp_keyfile_load(const char *path, void *dev_keys, uint64_t capacity,
                    uint64_t *count, int device, void *stream);
/* Device memory -> binary key file (D2H of chunk k+1 overlaps the write of
 * chunk k). */
int mp_keyfile_store(const char *path, const void *dev_keys, uint64_t count,
                     int device, void *stream);
/* File + file -> binary key file: the stable merge (MP_KEY_I64, ties to A)
 * of two sorted key files, i.e. dataio's read_keys on both inputs,
 * parallel_merge_into and write_keys_binary (dataio.cpp:33-98,
 * mergebench.cpp:243-259) as one call whose stages overlap.  Binary inputs
 * and the output are memory-mapped and streamed through mp_merge_host's
 * pipeline: page-cache reads, H2D copies, chunk merges, D2H copies and the
 * output's writes run concurrently.  Text inputs are parsed first.  *count
 * (optional) = keys written.  Blocks until the output file is complete.
 * The output must not be one of the inputs (MP_ERR_INVALID). */
int mp_keyfile_merge(const char *path_a, const char *path_b, const char *path_out,
                     uint64_t *count, int device);
/* File -> sorted binary key file (read_keys, parallel_merge_sort,
 * write_keys_binary: mergebench.cpp:326-332) through mp_sort_host's pipeline
 * on the mapped files. */
int mp_keyfile_sort(const char *path_in, const char *path_out, uint64_t *count,
                    int device);

#ifdef __cplusplus
}
#endif

#endif /* MERGEPATH_B200_H */
