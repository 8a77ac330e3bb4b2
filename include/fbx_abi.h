/* fbx_abi.h -- plain-C data layouts shared by the host runtime (libfbx.so),
 * the NVRTC-compiled plan kernels and the Python/ctypes host.
 *
 * No torch types, no C++: these structs cross the C-ABI and the kernel
 * parameter boundary unchanged.
 */
#ifndef FBX_ABI_H
#define FBX_ABI_H

#define FBX_ABI_VERSION 1
#define FBX_MAX_PARAM_SLOTS 384 /* u64 slots passed by value to a plan kernel */

/* Stage ranks of an error key (the reference's StageError.stage,
 * pipeline.py:96-104, in pipeline order). */
#define FBX_STAGE_PREPARE 0
#define FBX_STAGE_READ 1
#define FBX_STAGE_CLEAN 2
#define FBX_STAGE_JOIN 3
#define FBX_STAGE_EXTRACT 4
#define FBX_STAGE_MERGE 5
#define FBX_STAGE_EMIT 6

/* Error codes (low byte of an error key).  Mapped back to the reference's
 * exception types by the host (engine.py). */
#define FBX_ERR_NONE 0
#define FBX_ERR_TYPE 1            /* TypeError: mix/fold of str or float */
#define FBX_ERR_VALUE 2           /* ValueError: wrap_u64 of a negative, bad delimiter */
#define FBX_ERR_ENCODE 3          /* UnicodeEncodeError: lone surrogate reached UTF-8 */
#define FBX_ERR_POOL 4            /* PoolExhausted */
#define FBX_ERR_EMIT_NULL_LABEL 5 /* EmitError */
#define FBX_ERR_LABEL_RANGE 6     /* BatchInvariantError: label not 0/1 */
#define FBX_ERR_DUP_ID 7          /* MergeUniquenessError */
#define FBX_ERR_MULTI_MATCH 8     /* side view key matched >1 rows (dup ids after merge) */
#define FBX_ERR_JSON_BIGINT 9     /* ValueError: int literal > 4300 digits */
#define FBX_ERR_JSON_DEEP 10      /* unsupported: JSON nesting deeper than 64 */
#define FBX_ERR_UNICODE_LOWER 11  /* reserved: lower() is exact on device (Unicode 15 tables) */
#define FBX_ERR_FLOAT_OVERFLOW 12 /* OverflowError: float32 pack of a too-large value */
#define FBX_ERR_FLOAT_SLOWPATH 13 /* unsupported: inexact (>19 digit) decimal at a rounding tie */
#define FBX_ERR_INTERNAL 14       /* a plan invariant failed (never expected) */
#define FBX_ERR_POOL_KEY 15       /* unsupported: reference-arena order over Utf8 join keys */
#define FBX_ERR_BASIC_DUP 16      /* MergeUniquenessError: basic features repeat an instance id */

/* Device-resident run state: counters, the pool head, the error word.
 * One per engine, reset (error_key and the label positions = ~0, the rest 0)
 * before a run.  The (key, detail) pairs lead, 16-byte aligned: they are
 * updated together by one 128-bit CAS. */
typedef struct fbx_state {
  unsigned long long error_key;     /* min over failures (pipeline order) */
  unsigned long long error_detail;  /* ... and that failure's detail */
  unsigned long long emit_range_pos;   /* first emission position of a non-0/1 label */
  unsigned long long emit_range_label; /* ... and that label (MiniBatch.validate's message) */
  unsigned long long emit_null_pos;    /* first emission position of a null label */
  unsigned long long pool_flagged;  /* tiles whose reference ArenaPool demand may exceed
                                       pool_bytes: fbx_pool_account decides exactly */
  unsigned long long tile_ticket;   /* dynamic tile scheduler */
  unsigned long long pool_head;     /* bump pointer of the HBM arena */
  unsigned long long pool_overflow; /* device arena too small: the head this launch needed
                                       (the engine grows the arena and re-runs) */
  unsigned long long digest;        /* XOR of instance digests */
  unsigned long long instances;
  unsigned long long signs;
  unsigned long long malformed;     /* CleanCounters.malformed_rows */
  unsigned long long filtered;      /* CleanCounters.filtered_rows */
  unsigned long long joined;        /* rows surviving the join(s) */
  unsigned long long side_rows;     /* side-view rows indexed */
  unsigned long long dup_seen;      /* an instance id was inserted twice (resolved by
                                       fbx_dup_resolve to the reference's chunk) */
  unsigned long long pad;
} fbx_state;

/* One device-placed pool-consuming operator node (reference: token pre/post
 * calls placed on the device, featureops.py:392-412, device.py:328-338), in the
 * order the reference runs them: layer, then name within the layer. */
typedef struct fbx_pool_node {
  unsigned int layer; /* 1-based layer */
  unsigned int rank;  /* node rank of the error key */
  unsigned int input; /* plane of the per-row lane sizes */
  unsigned int pad;
} fbx_pool_node;

/* Kernel parameter block: program-defined u64 slots (device pointers, sizes,
 * row ranges).  The planner that generated the program assigns the slots. */
typedef struct fbx_params {
  unsigned long long v[FBX_MAX_PARAM_SLOTS];
} fbx_params;

#endif /* FBX_ABI_H */
