/* fbx.h -- C-ABI of libfbx.so, the B200 FeatureBox extraction runtime.
 *
 * Replaces, for the per-record extraction path, the reference's
 *   pipeline._extract_batch(table, prepared, ctx)   pkg/src/featurebox/pipeline.py:718-737
 *   device.execute_plan(ctx, plan, dag, state, ev)  pkg/src/featurebox/device.py:434-444
 *   device.NodeEvaluator.__init__ (resolve + bind)  pkg/src/featurebox/device.py:263-293
 *   mempool.ArenaPool / group_allocate / reset      pkg/src/featurebox/mempool.py:87-145
 *   featureops.DictTable / dict_lookup              pkg/src/featurebox/featureops.py:104-167
 *   viewpipe.JoinIndex / join_with_index (probe)    pkg/src/featurebox/viewpipe.py:498-547
 *
 * All entry points take plain pointers and sizes.  Every function returns 0
 * on success or a negative FBX_E* code; fbx_last_error() gives the message
 * (thread-local).  Device pointers are CUDA device addresses; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Calls release no locks of
 * their own and are safe to call from a thread without the Python GIL.
 */
#ifndef FBX_H
#define FBX_H

#include <stddef.h>
#include <stdint.h>

#include "fbx_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FBX_OK 0
#define FBX_E_ARG (-1)
#define FBX_E_COMPILE (-2)
#define FBX_E_CUDA (-3)
#define FBX_E_NOT_FOUND (-4)
#define FBX_E_DUPLICATE (-5)
#define FBX_E_IO (-6)

typedef struct fbx_program fbx_program; /* a loaded plan module (CUmodule) */
typedef struct fbx_kernel fbx_kernel;   /* one kernel of a program */

const char* fbx_version(void);

/* -- plan compilation (host-only; no GPU needed) ------------------------
 * Compile a generated plan source (NVRTC, -arch=sm_100a) to a cubin.
 * Replaces NodeEvaluator's once-per-run resolution (device.py:271-293) and
 * the paper's runtime-compiled meta-kernel.  *image is
 * malloc'ed; free with fbx_free(). */
int fbx_compile(const char* source, const char* program_name, const char* const* options,
                int n_options, void** image, size_t* image_bytes, char* log, size_t log_capacity);
void fbx_free(void* p);

/* -- program loading / launching (needs a GPU) -------------------------- */
int fbx_program_load(const void* image, size_t image_bytes, fbx_program** out);
int fbx_program_unload(fbx_program* prog);
int fbx_program_kernel(fbx_program* prog, const char* name, fbx_kernel** out);
/* max dynamic shared memory / register info of a kernel */
int fbx_kernel_attributes(fbx_kernel* k, int* num_regs, int* max_threads, int* static_smem);
int fbx_kernel_set_max_dynamic_smem(fbx_kernel* k, int bytes);

/* Launch one plan kernel.  The layered operator DAG of a whole driver chunk
 * runs inside this one launch (execute_plan's per-layer barriers become the
 * per-row program order, since every operator is row-local). */
int fbx_launch(fbx_kernel* k, unsigned grid, unsigned block, unsigned dyn_smem, void* stream,
               const fbx_params* params);

/* -- arena + state helpers ---------------------------------------------- */
/* Reset the run state (counters, pool head, error word, tile ticket) and the
 * per-tile look-back status words: mempool.ArenaPool.reset (mempool.py:136). */
int fbx_state_reset(fbx_state* d_state, unsigned long long* d_tile_status, size_t n_tiles,
                    void* stream);

/* Clear check_unique_ids' run-wide id set (viewpipe.py:562-576 `seen`, pipeline.py:
 * 1071) for a new run, and its later-occurrence pairs only when the previous run's
 * state says an id repeated (decided on the device; call BEFORE fbx_state_reset). */
int fbx_idset_clear(unsigned long long* d_ids, size_t n_words, unsigned long long* d_pairs,
                    size_t n_pair_words, const fbx_state* d_state, void* stream);

/* The reference ArenaPool's PoolExhausted for the chunks a plan kernel flagged
 * (state.pool_flagged != 0): one CTA per chunk ranks the chunk's joined rows by
 * join-key image, sums each device token node's lane sizes per group of
 * lanes_per_group rows and walks the grants against `capacity` with the head
 * reset per layer (mempool.py:114-134, device.py:181-196, 328-338, 408-409);
 * the first grant past capacity is raised as FBX_ERR_POOL at (chunk, layer,
 * node) with detail (requested << 32) | remaining.  Scratch: n_tiles*tile_rows
 * u32 + u64. */
int fbx_pool_account(const unsigned char* d_tile_flag, const unsigned long long* d_tile_chunk,
                     unsigned long long n_tiles, unsigned spc, unsigned tile_rows,
                     const unsigned long long* d_keys, unsigned kw, const unsigned* d_sizes,
                     unsigned ni, const unsigned char* d_joined, const fbx_pool_node* d_nodes,
                     unsigned n_nodes, unsigned long long lanes_per_group,
                     unsigned long long capacity, unsigned* d_rank_scratch,
                     unsigned long long* d_sum_scratch, fbx_state* d_state, void* stream);

/* cudaMemsetAsync on `stream` (zeroing the hash tables before an index rebuild). */
int fbx_memset_async(void* d_ptr, int value, size_t bytes, void* stream);

/* Reset the per-launch part of the run state -- the bump-pool head (ArenaPool.reset,
 * mempool.py:136) and the persistent kernel's tile ticket -- between the launches of
 * one run, whose counters keep accumulating. */
int fbx_pool_reset(fbx_state* d_state, void* stream);

/* Copy the run state (fbx_state) into host-mapped pinned memory with a kernel on
 * `stream` (no copy engine: the snapshot never waits behind bulk D2H transfers).
 * Streamed runs read each slice's emitted counts from it to size the CSR D2H.
 * Replaces the per-batch counter read of device.py:110-113 / pipeline.py:883-886. */
int fbx_state_snapshot(const fbx_state* d_state, void* h_mapped_dst, void* stream);

/* Build an HBM open-addressing dictionary table (featureops.py:104-167):
 * n keys given as a byte blob + u32 offsets[n+1] (device), u64 values.
 * slots: capacity * 32 bytes (capacity a power of two >= 2n).  Returns
 * FBX_E_DUPLICATE when two keys are equal (load_dict_table's duplicate-key
 * error, featureops.py:147). */
int fbx_dict_build(void* d_slots, unsigned long long capacity, const unsigned char* d_keyblob,
                   const unsigned int* d_key_offsets, const unsigned long long* d_values,
                   unsigned long long n, unsigned long long* d_dup_flag, void* stream);

/* Row-aligned string outputs of the _extract_batch kernel (pipeline.py:731-736):
 * out[0] = 0, out[i+1] = in[0] + ... + in[i]  (u32 lengths -> u64 FBXC offsets) */
int fbx_exclusive_scan_u32(const unsigned int* d_in, unsigned long long* d_out,
                           unsigned long long n, void* stream);
/* Copy n pool-resident strings (pointer, length) into one FBXC data segment. */
int fbx_gather_strings(const unsigned long long* d_ptrs, const unsigned int* d_lens,
                       const unsigned long long* d_offsets, unsigned long long n,
                       unsigned char* d_out, void* stream);

/* check_unique_ids' failing row (viewpipe.py:562-576 as called at
 * pipeline.py:1071): the row of an instance id's SECOND occurrence in row
 * order, minimised over ids (its chunk is row / batch_size).  d_winner_row[i] is
 * the row that claimed id-set slot i, d_later_rows[2i], [2i+1] the two smallest
 * rows (stored as ~row, 0 = none) that found the id already present.  Writes the answer row
 * to d_out[0] and its slot to d_out[1] (~0 when no id repeats). */
int fbx_dup_resolve(const unsigned long long* d_winner_row,
                    const unsigned long long* d_later_rows, unsigned long long n_slots,
                    unsigned long long* d_out, void* stream);

/* Write `bytes` of a scratch buffer (an L2 flush between timed steps). */
/* zlib CRC-32 of n device bytes into *d_out (columnstore.py:554-562: the FBXC body
 * check of a full read, done where the body already is -- in HBM).  d_scratch holds
 * fbx_crc32_scratch_words(n) words.  Two launches on `stream`, no host sync. */
int fbx_crc32(const void* d_buf, unsigned long long n, unsigned* d_scratch, unsigned* d_out,
              void* stream);
unsigned long long fbx_crc32_scratch_words(unsigned long long n);

int fbx_l2_flush(void* d_buf, size_t bytes, void* stream);

/* batch_size > 1024 (a chunk cut into 512-row sub-tiles): the n
 * instances of a range, emitted as spc sorted runs per chunk, re-ordered into
 * each chunk's ascending-id order (emit order, viewpipe.py:521) with their
 * (slot, sign) segments -- the CSR of d_ids/d_lab/d_off[n+1]/d_slot/d_sign
 * (offsets absolute, the range's signs start at s0) written to the _o arrays.
 * d_tile_start[n_tiles+1]: first instance of every sub-tile relative to the
 * range.  d_scratch: 3n+1 words.  *d_bad set (nothing written) when a length
 * is outside [0, max_len] -- only a failing run's CSR (repeated id). */
int fbx_merge_subtiles(const unsigned long long* d_tile_start, unsigned spc,
                       unsigned long long n_tiles, unsigned long long n, unsigned long long s0,
                       unsigned max_len, const unsigned long long* d_ids,
                       const unsigned char* d_lab, const unsigned long long* d_off,
                       const unsigned short* d_slot, const unsigned long long* d_sign,
                       unsigned long long* d_ids_o, unsigned char* d_lab_o,
                       unsigned long long* d_off_o, unsigned short* d_slot_o,
                       unsigned long long* d_sign_o, unsigned long long* d_scratch,
                       unsigned* d_bad, void* stream);

/* Whole-table operations of the staged mode (pipeline.run_staged,
 * pipeline.py:783-895; csrc/fbx_table.cu).  Keys: the u64 whose unsigned order
 * is the reference key image's order (join_key_bytes, viewpipe.py:451-459):
 * Int64 two's-complement bits, Float32 IEEE bits. */
/* clean_views' survivors: indices of the rows with keep[i] != 0, in order. */
int fbx_select_rows(const unsigned char* d_keep, unsigned long long n, unsigned* d_rows,
                    unsigned long long* d_count, void* stream);
/* dst[i] = src[rows[i]] for elements of 1, 2, 4 or 8 bytes. */
int fbx_take(const void* d_src, unsigned elem_bytes, const unsigned* d_rows,
             unsigned long long n, void* d_dst, void* stream);
/* FBXC null bitmap (LSB-first, set = null) of rows[i] (or i when rows is NULL). */
int fbx_pack_nulls(const unsigned char* d_isnull, const unsigned* d_rows, unsigned long long n,
                   unsigned char* d_bitmap, void* stream);
/* Per-row null bytes of an FBXC bitmap; (pointer, length) of every string of a
 * Utf8 / Json image (offsets[n+1] into data). */
int fbx_unpack_nulls(const unsigned char* d_bitmap, unsigned long long n,
                     unsigned char* d_isnull, void* stream);
int fbx_spans(const unsigned* d_offsets, const unsigned char* d_data, unsigned long long n,
              unsigned long long* d_ptr, unsigned* d_len, void* stream);
/* JoinIndex (viewpipe.py:498-511): the non-null keys and their rows, sorted by key
 * (stable); *d_count = how many.  Scratch: n rows, n keys, n flag bytes. */
int fbx_sort_keys(const unsigned long long* d_key, const unsigned char* d_isnull,
                  unsigned long long n, unsigned long long* d_skey, unsigned* d_srow,
                  unsigned long long* d_count, unsigned* d_rows_scratch,
                  unsigned long long* d_key_scratch, unsigned char* d_flag_scratch, void* stream);
/* join_with_index (viewpipe.py:537-547): matches per left row (first sorted index,
 * count); the host scans the counts into offsets, then fbx_join_fill writes the
 * m matches' (left row, right row) in _materialize_join's (key, left, right) order. */
int fbx_join_count(const unsigned long long* d_lkey, const unsigned char* d_lnull,
                   unsigned long long nl, const unsigned long long* d_skey,
                   unsigned long long nr_valid, unsigned long long* d_first, unsigned* d_cnt,
                   void* stream);
int fbx_join_fill(const unsigned long long* d_lkey, unsigned long long nl,
                  const unsigned long long* d_first, const unsigned* d_cnt,
                  const unsigned long long* d_off, const unsigned* d_srow, unsigned long long m,
                  unsigned* d_left, unsigned* d_right, void* stream);
/* check_unique_ids (viewpipe.py:562-576) over sorted keys: the first row, in row
 * order, whose key occurred before (~0 when none). */
int fbx_first_repeat(const unsigned long long* d_skey, const unsigned* d_srow,
                     unsigned long long n_valid, unsigned long long* d_best, void* stream);
/* check_unique_ids across the record shards of one log (sharded.py).
 * fbx_idset_entries: every id the engine's run-wide id set holds (slots
 * [0, cap) keyed by the id, slot cap = id 0) with the first row holding it --
 * the smaller of the slot's winner row and its smallest later row (~row coded);
 * *d_count = how many (order unspecified).  Buffers: cap + 1 entries. */
int fbx_idset_entries(const unsigned long long* d_set, const unsigned long long* d_win_rows,
                      const unsigned long long* d_later_rows, unsigned long long cap,
                      unsigned long long* d_ids, unsigned long long* d_rows,
                      unsigned long long* d_count, void* stream);
/* The first row (smallest d_rows entry) whose id is in d_prior (the ids of the
 * lower shards, any order): d_out[0] = that row, d_out[1] = its id; both ~0
 * when none.  Replaces the reference's `seen` set carried across chunks
 * (pipeline.py:1071-1072, viewpipe.py:562-576) at a shard boundary. */
int fbx_seen_before(const unsigned long long* d_ids, const unsigned long long* d_rows,
                    unsigned long long n, const unsigned long long* d_prior,
                    unsigned long long n_prior, unsigned long long* d_out, void* stream);

/* Host ingest of a driver slice (read_columns with a row range,
 * columnstore.py:499-608; pipeline.py:986-1006 reads the driver chunk by chunk):
 * n_spans byte spans of one FBXC file, span i = file bytes
 * [file_off[i], file_off[i] + len[i]) -> dst + dst_off[i].  pread(2) from a pool
 * of n_threads host threads (1 MiB pieces) straight into the (pinned) staging
 * buffer that the H2D copy reads next.  FBX_E_IO on an open / read failure or a
 * span past the end of the file (the reference's TruncatedError). */
int fbx_read_spans(const char* path, void* dst, const unsigned long long* file_off,
                   const unsigned long long* len, const unsigned long long* dst_off,
                   unsigned n_spans, unsigned n_threads);

/* =======================================================================
 * The engine object: the drop-in for the reference's extraction boundary
 * (SURVEY.md §8 b).
 *
 *   fbx_create      NodeEvaluator.__init__ + ExecContext     device.py:99-149, 263-293
 *                   (plan bound once, tables built in HBM)   featureops.py:104-167
 *   fbx_extract     pipeline._extract_batch(table, prep, ctx) pipeline.py:718-737
 *                   = execute_plan over the layered DAG       device.py:434-444
 *                   counters as ExecContext's                 device.py:110-113
 *   fbx_output_*    the appended output columns (count pass, then copy)
 *   fbx_emit_csr    emit_minibatch + MiniBatch.validate +     pipeline.py:357-433
 *                   instance_digest / batch_digest
 *   fbx_last_error  LayerExecutionError(layer, node, cause)   device.py:34-41
 *   fbx_destroy
 *
 * Columns cross as FBXC images (fbxc_format.md:68-126): a null bitmap
 * (LSB-first, set = null), int64[n] / float32[n] payloads or u32 offsets[n+1]
 * + UTF-8 bytes.  Input and output pointers may be host (pageable or pinned)
 * or device memory: the engine stages through its own HBM buffers.  One
 * engine per GPU and per calling thread; calls do not touch the Python GIL.
 * ======================================================================= */

/* fbx_extract / fbx_emit_csr status: the reference exception they stand for */
#define FBX_S_OK 0
#define FBX_S_CONFIG 1         /* ConfigError / FeatureConfigError */
#define FBX_S_POOL_EXHAUSTED 2 /* PoolExhausted(requested, remaining) */
#define FBX_S_TYPE 3           /* TypeError (mix / fold of str or float) */
#define FBX_S_VALUE 4          /* ValueError (wrap_u64 of a negative, bad delimiter, ...) */
#define FBX_S_ENCODE 5         /* UnicodeEncodeError (lone surrogate) */
#define FBX_S_CUDA 6           /* CUDA failure */
#define FBX_S_OVERFLOW 7       /* OverflowError (float32 pack) */
#define FBX_S_UNSUPPORTED 8    /* a row needs a path the device does not implement */
#define FBX_S_EMIT 9           /* EmitError (null instance id / label at emission) */
#define FBX_S_INVARIANT 10     /* BatchInvariantError (duplicate id, label not 0/1) */
#define FBX_S_INTERNAL 11

#define FBX_KIND_INT64 0
#define FBX_KIND_FLOAT32 1
#define FBX_KIND_UTF8 2
#define FBX_KIND_JSON 3

typedef struct fbx_engine fbx_engine;

typedef struct fbx_column {
  unsigned int kind;              /* FBX_KIND_* */
  const unsigned char* nulls;     /* (n+7)/8 bytes */
  const void* data;               /* int64[n] | float32[n] | data_bytes UTF-8 bytes */
  const unsigned int* offsets;    /* var-length kinds: n+1 */
  unsigned long long data_bytes;  /* var-length kinds: offsets[n] */
} fbx_column;

/* A plan as the host planner emits it: the compiled row-aligned extraction
 * kernel (fbx_compile of the generated source) and its parameter-slot map.
 * Slot -1 = unused. */
typedef struct fbx_plan {
  const void* cubin;
  size_t cubin_bytes;
  const char* kernel;                  /* "fbx_extract_rows" */
  int slot_state, slot_rows, slot_pool, slot_pool_cap, slot_pool_sizes;
  unsigned int n_inputs;               /* table columns, in fbx_extract's order */
  const unsigned int* input_kinds;     /* [n_inputs] */
  const int* input_slots;              /* [n_inputs][3]: nulls, data, offsets */
  unsigned int n_outputs;              /* appended columns, in output order */
  const unsigned int* output_kinds;    /* [n_outputs]: FBX_KIND_INT64 | FBX_KIND_UTF8 */
  const int* output_slots;             /* [n_outputs][4]: nulls, data, ptr, len */
  unsigned int n_tables;
  const int* table_slots;              /* [n_tables][3]: slots, mask, keys */
  unsigned int n_pool_nodes;           /* device token nodes, reference order */
  const fbx_pool_node* pool_nodes;
  unsigned int pool_planes;
  unsigned long long pool_bytes;       /* config device.pool_bytes */
  unsigned long long lanes_per_group;  /* config device.lanes_per_group */
  unsigned int n_nodes;                /* every DAG node, error-rank order */
  const char* const* node_names;
  unsigned long long arena_bytes_per_row; /* initial device arena (grown on demand) */
} fbx_plan;

/* One dictionary (featureops.DictTable): keys as a byte blob + u32 offsets[n+1],
 * u64 values; host or device memory. */
typedef struct fbx_table {
  const unsigned char* keys;
  const unsigned int* key_offsets;
  const unsigned long long* values;
  unsigned long long n;
} fbx_table;

typedef struct fbx_counters {      /* ExecContext counters (device.py:110-113) */
  unsigned long long launches;     /* kernels launched by the call */
  unsigned long long rows;
  unsigned long long bytes_h2d;    /* input bytes staged from host memory */
  double device_ms;                /* CUDA-event time of the extraction kernels */
} fbx_counters;

typedef struct fbx_csr {           /* caller buffers (host or device) */
  unsigned long long* ids;         /* n   (u64 image of the instance id) */
  unsigned char* labels;           /* n */
  unsigned long long* offsets;     /* n+1 */
  unsigned short* slots;           /* capacity */
  unsigned long long* signs;       /* capacity */
  unsigned long long capacity;     /* sign slots available; 0 = count pass only */
  unsigned long long n_signs;      /* out: signs of the batch */
  unsigned long long digest;       /* out: batch_digest (XOR of instance digests) */
} fbx_csr;

int fbx_create(const fbx_plan* plan, const fbx_table* tables, int device, fbx_engine** out);
int fbx_destroy(fbx_engine* e);

/* Run the plan over n_rows rows of the table (columns in plan input order).
 * Returns FBX_S_* (the reference's failure, located by fbx_last_error) or a
 * negative FBX_E_* for a misuse.  Outputs stay in the engine until the next
 * call. */
int fbx_extract(fbx_engine* e, const fbx_column* cols, unsigned int n_cols,
                unsigned long long n_rows, fbx_counters* counters, void* stream);
/* Output j of the last fbx_extract: its kind and payload byte count (count pass). */
int fbx_output_info(const fbx_engine* e, unsigned int j, unsigned int* kind,
                    unsigned long long* n_rows, unsigned long long* data_bytes);
/* Copy output j into caller buffers: nulls (n+7)/8 bytes, data (int64[n] or
 * data_bytes), offsets u32[n+1] (var-length only). */
int fbx_output_copy(fbx_engine* e, unsigned int j, unsigned char* nulls, void* data,
                    unsigned int* offsets, void* stream);

/* emit_minibatch over n rows: per row the non-null features as (slot, sign)
 * pairs, deduplicated and sorted; ids / labels; the batch digest.  Fails like
 * the reference: FBX_S_EMIT for the first null id or label, FBX_S_INVARIANT for
 * a duplicate id or a label outside {0, 1} (MiniBatch.validate).  Call with
 * capacity 0 to size the sign buffers (n_signs). */
int fbx_emit_csr(fbx_engine* e, const fbx_column* ids, const fbx_column* labels,
                 const fbx_column* features, const unsigned int* slots, unsigned int k,
                 unsigned long long n_rows, fbx_csr* out, void* stream);

/* The last call's failure: returns its FBX_S_* status and sets *layer (0 when
 * not an operator failure), *node (node name or NULL) and, when non-NULL,
 * *detail (PoolExhausted: requested << 32 | remaining; emit: the row). */
int fbx_last_error(const fbx_engine* e, int* layer, const char** node,
                   unsigned long long* detail);
/* Human-readable message of the last failure of e, or (e == NULL) of the
 * calling thread's last API error. */
const char* fbx_error_message(const fbx_engine* e);

#ifdef __cplusplus
}
#endif

#endif /* FBX_H */
