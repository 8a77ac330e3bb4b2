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

typedef struct fbx_program fbx_program; /* a loaded plan module (CUmodule) */
typedef struct fbx_kernel fbx_kernel;   /* one kernel of a program */

const char* fbx_version(void);
const char* fbx_last_error(void);

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

/* check_unique_ids' failing chunk (viewpipe.py:562-576 as called at
 * pipeline.py:1071): the chunk of an instance id's SECOND occurrence in chunk
 * order, minimised over ids.  d_winner_chunk[i] is the chunk of the row that
 * claimed id-set slot i, d_later_chunks[i] the two smallest chunks (+1, packed
 * hi|lo, 0 = none) of the rows that found the id already present.  Writes
 * (chunk << 32 | slot) of the answer to *d_out, ~0 when no id repeats. */
int fbx_dup_resolve(const unsigned int* d_winner_chunk, const unsigned long long* d_later_chunks,
                    unsigned long long n_slots, unsigned long long* d_out, void* stream);

/* Write `bytes` of a scratch buffer (an L2 flush between timed steps). */
/* zlib CRC-32 of n device bytes into *d_out (columnstore.py:554-562: the FBXC body
 * check of a full read, done where the body already is -- in HBM).  d_scratch holds
 * fbx_crc32_scratch_words(n) words.  Two launches on `stream`, no host sync. */
int fbx_crc32(const void* d_buf, unsigned long long n, unsigned* d_scratch, unsigned* d_out,
              void* stream);
unsigned long long fbx_crc32_scratch_words(unsigned long long n);

int fbx_l2_flush(void* d_buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FBX_H */
