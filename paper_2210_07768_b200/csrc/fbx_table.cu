// fbx_table.cu -- libfbx.so: whole-table operations of the staged mode
// (pipeline.run_staged, pipeline.py:783-895), on the device.
//
// The staged mode materialises every stage boundary as an FBXC file; its
// table operations are the reference's viewpipe ones applied to whole tables:
//
//   fbx_select_rows   the survivors of clean_views (viewpipe.py:334-431):
//                     stream compaction of a keep mask into row indices
//   fbx_take          a column's values at those rows (any element width)
//   fbx_pack_nulls    an FBXC null bitmap (LSB-first, set = null) from per-row bytes
//   fbx_unpack_nulls  the reverse; fbx_spans: (pointer, length) of every string
//   fbx_sort_keys     the right side of a join (JoinIndex, viewpipe.py:498-511):
//                     the non-null keys and their rows, sorted by key (stable, so
//                     equal keys keep row order)
//   fbx_join_count /  join_with_index (viewpipe.py:537-547) + _materialize_join's
//   fbx_join_fill     sort (:514-534): every (left row, right row) match, in
//                     (key image, left row, right row) order
//   fbx_first_repeat  check_unique_ids (viewpipe.py:562-576): the first row, in row
//                     order, whose id occurred before
//   fbx_idset_entries / fbx_seen_before
//                     check_unique_ids across the record shards of one log
//                     (sharded.py): every id a shard's run inserted with the
//                     first row holding it; the first of them, in row order,
//                     that a lower shard holds
//
// Keys are given as the u64 whose unsigned order is the order of the reference's
// key image (join_key_bytes, viewpipe.py:451-459: kind tag, length, big-endian
// payload): an Int64 key is its two's-complement bits, a Float32 key its IEEE
// bits -- the big-endian bytes of both compare as the unsigned integer.

#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <string>

#include "fbx.h"

extern "C" int fbx_internal_fail(int code, const char* msg);

namespace {

typedef unsigned long long ull;

int tcheck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FBX_OK;
  return fbx_internal_fail(FBX_E_CUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

unsigned grid_for(ull n) {
  const ull b = (n + 255) / 256;
  return (unsigned)(b < 4736 ? (b ? b : 1) : 4736);
}

template <typename T>
__global__ void k_take(const T* src, const unsigned* idx, ull n, T* dst) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// one warp packs 32 rows into 4 bitmap bytes (ballot); n rows, bytes ceil(n/8)
__global__ void k_pack_nulls(const unsigned char* isnull, const unsigned* idx, ull n,
                             unsigned char* bitmap) {
  const ull warps = ((ull)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  for (ull w = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 < n; w += warps) {
    const ull i = w * 32 + lane;
    const bool nl = i < n && isnull[idx ? idx[i] : i] != 0;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, nl);
    if (lane < 4u && w * 32 + lane * 8 < n) bitmap[w * 4 + lane] = (unsigned char)(b >> (8 * lane));
  }
}

__global__ void k_unpack_nulls(const unsigned char* bitmap, ull n, unsigned char* isnull) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x)
    isnull[i] = (bitmap[i >> 3] >> (i & 7u)) & 1u;
}

__global__ void k_spans(const unsigned* offsets, const unsigned char* data, ull n, ull* ptr,
                        unsigned* len) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x) {
    ptr[i] = (ull)(data + offsets[i]);
    len[i] = offsets[i + 1] - offsets[i];
  }
}

__global__ void k_valid_flags(const unsigned char* isnull, ull n, unsigned char* flag) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x)
    flag[i] = isnull ? (unsigned char)(isnull[i] == 0) : (unsigned char)1;
}

// slots past the valid count: the largest key and row ~0 -- they sort last (a
// valid key equal to ~0 stays before them: the radix sort is stable)
__global__ void k_gather_keys(const ull* key, unsigned* rows, ull n, const ull* count, ull* out) {
  const ull c = *count;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x) {
    if (i < c) {
      out[i] = key[rows[i]];
    } else {
      out[i] = ~0ull;
      rows[i] = 0xFFFFFFFFu;
    }
  }
}

__global__ void k_iota(unsigned* a, ull n) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x)
    a[i] = (unsigned)i;
}

__device__ __forceinline__ ull lower_bound_u64(const ull* a, ull n, ull k) {
  ull lo = 0, hi = n;
  while (lo < hi) {
    const ull m = (lo + hi) >> 1;
    if (a[m] < k) lo = m + 1; else hi = m;
  }
  return lo;
}

__global__ void k_join_count(const ull* lkey, const unsigned char* lnull, ull nl, const ull* skey,
                             ull nr, ull* first, unsigned* cnt) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (ull)gridDim.x * blockDim.x) {
    if (lnull && lnull[i]) {
      first[i] = 0;
      cnt[i] = 0;
      continue;
    }
    const ull k = lkey[i];
    const ull a = lower_bound_u64(skey, nr, k);
    ull b = a;
    while (b < nr && skey[b] == k) ++b;  // matches of one key (unique on the merge side)
    first[i] = a;
    cnt[i] = (unsigned)(b - a);
  }
}

__global__ void k_join_fill(const ull* lkey, ull nl, const ull* first, const unsigned* cnt,
                            const ull* off, const unsigned* srow, ull* pkey, unsigned* pl,
                            unsigned* pr) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (ull)gridDim.x * blockDim.x) {
    const ull o = off[i];
    for (unsigned j = 0; j < cnt[i]; ++j) {
      pkey[o + j] = lkey[i];
      pl[o + j] = (unsigned)i;
      pr[o + j] = srow[first[i] + j];
    }
  }
}

__global__ void k_first_repeat(const ull* skey, const unsigned* srow, ull n, ull* best) {
  for (ull p = (ull)blockIdx.x * blockDim.x + threadIdx.x + 1; p < n; p += (ull)gridDim.x * blockDim.x)
    if (skey[p] == skey[p - 1]) atomicMin(best, (ull)srow[p]);
}

// the engine's run-wide id set (codegen ids tail): slots [0, cap) keyed by the
// id, slot cap = id 0 (stored as 1); the winner's row per slot and the two
// smallest later rows (as ~row, 0 = none)
__global__ void k_idset_entries(const ull* set, const ull* win, const ull* later, ull cap,
                                ull* ids, ull* rows, ull* count) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i <= cap; i += (ull)gridDim.x * blockDim.x) {
    const ull v = set[i];
    if (v == 0ull) continue;
    ull r = win[i];
    const ull x = later[2 * i];  // ~(smallest later row), 0 = none
    if (x && ~x < r) r = ~x;
    const ull k = atomicAdd(count, 1ull);
    ids[k] = i == cap ? 0ull : v;
    rows[k] = r;
  }
}

__global__ void k_seen_before(const ull* ids, const ull* rows, ull n, const ull* prior, ull np,
                              ull* best) {
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x) {
    const ull k = ids[i];
    const ull a = lower_bound_u64(prior, np, k);
    if (a < np && prior[a] == k) atomicMin(best, rows[i]);
  }
}

__global__ void k_seen_before_id(const ull* ids, const ull* rows, ull n, ull* best) {
  const ull b = best[0];
  if (b == ~0ull) return;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (ull)gridDim.x * blockDim.x)
    if (rows[i] == b) best[1] = ids[i];  // one entry per row: a row holds one id
}

template <typename F>
int with_temp(size_t bytes, cudaStream_t s, F&& f) {
  void* tmp = nullptr;
  int rc = tcheck(cudaMallocAsync(&tmp, bytes ? bytes : 16, s), "table temp");
  if (rc) return rc;
  f(tmp);
  rc = tcheck(cudaGetLastError(), "table op");
  cudaFreeAsync(tmp, s);
  return rc;
}

}  // namespace

extern "C" {

int fbx_select_rows(const unsigned char* d_keep, unsigned long long n, unsigned* d_rows,
                    unsigned long long* d_count, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = tcheck(cudaMemsetAsync(d_count, 0, sizeof(ull), s), "select count");
  if (rc || n == 0) return rc;
  thrust::counting_iterator<unsigned> it(0u);
  size_t bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, bytes, it, d_keep, d_rows, d_count, (int)n, s);
  return with_temp(bytes, s, [&](void* t) {
    cub::DeviceSelect::Flagged(t, bytes, it, d_keep, d_rows, d_count, (int)n, s);
  });
}

int fbx_take(const void* d_src, unsigned elem_bytes, const unsigned* d_rows,
             unsigned long long n, void* d_dst, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return FBX_OK;
  const unsigned g = grid_for(n);
  switch (elem_bytes) {
    case 1: k_take<<<g, 256, 0, s>>>((const unsigned char*)d_src, d_rows, n, (unsigned char*)d_dst); break;
    case 2: k_take<<<g, 256, 0, s>>>((const unsigned short*)d_src, d_rows, n, (unsigned short*)d_dst); break;
    case 4: k_take<<<g, 256, 0, s>>>((const unsigned*)d_src, d_rows, n, (unsigned*)d_dst); break;
    case 8: k_take<<<g, 256, 0, s>>>((const ull*)d_src, d_rows, n, (ull*)d_dst); break;
    default: return fbx_internal_fail(FBX_E_ARG, "fbx_take: element of 1, 2, 4 or 8 bytes");
  }
  return tcheck(cudaGetLastError(), "fbx_take");
}

int fbx_pack_nulls(const unsigned char* d_isnull, const unsigned* d_rows, unsigned long long n,
                   unsigned char* d_bitmap, void* stream) {
  if (n == 0) return FBX_OK;
  k_pack_nulls<<<grid_for((n + 7) / 8 * 8), 256, 0, (cudaStream_t)stream>>>(d_isnull, d_rows, n,
                                                                           d_bitmap);
  return tcheck(cudaGetLastError(), "fbx_pack_nulls");
}

int fbx_unpack_nulls(const unsigned char* d_bitmap, unsigned long long n,
                     unsigned char* d_isnull, void* stream) {
  if (n == 0) return FBX_OK;
  k_unpack_nulls<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_bitmap, n, d_isnull);
  return tcheck(cudaGetLastError(), "fbx_unpack_nulls");
}

int fbx_spans(const unsigned* d_offsets, const unsigned char* d_data, unsigned long long n,
              unsigned long long* d_ptr, unsigned* d_len, void* stream) {
  if (n == 0) return FBX_OK;
  k_spans<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_offsets, d_data, n, d_ptr, d_len);
  return tcheck(cudaGetLastError(), "fbx_spans");
}

int fbx_sort_keys(const unsigned long long* d_key, const unsigned char* d_isnull,
                  unsigned long long n, unsigned long long* d_skey, unsigned* d_srow,
                  unsigned long long* d_count, unsigned* d_rows_scratch,
                  unsigned long long* d_key_scratch, unsigned char* d_flag_scratch, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = tcheck(cudaMemsetAsync(d_count, 0, sizeof(ull), s), "sort count");
  if (rc || n == 0) return rc;
  k_valid_flags<<<grid_for(n), 256, 0, s>>>(d_isnull, n, d_flag_scratch);
  rc = fbx_select_rows(d_flag_scratch, n, d_rows_scratch, d_count, stream);
  if (rc) return rc;
  // sort all n slots: the first *d_count are the valid keys (read by the caller)
  k_gather_keys<<<grid_for(n), 256, 0, s>>>(d_key, d_rows_scratch, n, d_count, d_key_scratch);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, d_key_scratch, d_skey, d_rows_scratch, d_srow,
                                  (int)n, 0, 64, s);
  return with_temp(bytes, s, [&](void* t) {
    cub::DeviceRadixSort::SortPairs(t, bytes, d_key_scratch, d_skey, d_rows_scratch, d_srow,
                                    (int)n, 0, 64, s);
  });
}

int fbx_join_count(const unsigned long long* d_lkey, const unsigned char* d_lnull,
                   unsigned long long nl, const unsigned long long* d_skey,
                   unsigned long long nr_valid, unsigned long long* d_first, unsigned* d_cnt,
                   void* stream) {
  if (nl == 0) return FBX_OK;
  k_join_count<<<grid_for(nl), 256, 0, (cudaStream_t)stream>>>(d_lkey, d_lnull, nl, d_skey,
                                                               nr_valid, d_first, d_cnt);
  return tcheck(cudaGetLastError(), "fbx_join_count");
}

int fbx_join_fill(const unsigned long long* d_lkey, unsigned long long nl,
                  const unsigned long long* d_first, const unsigned* d_cnt,
                  const unsigned long long* d_off, const unsigned* d_srow, unsigned long long m,
                  unsigned* d_left, unsigned* d_right, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (m == 0) return FBX_OK;
  // the matches in (left row, right row) order, then a stable radix sort by key
  // image: (key, left row, right row), _materialize_join's matches.sort()
  ull *pkey = nullptr;
  unsigned* pw = nullptr;
  int rc = tcheck(cudaMallocAsync((void**)&pkey, 2 * m * sizeof(ull), s), "join keys");
  if (rc) return rc;
  rc = tcheck(cudaMallocAsync((void**)&pw, 4 * m * sizeof(unsigned), s), "join rows");
  if (rc) {
    cudaFreeAsync(pkey, s);
    return rc;
  }
  unsigned *pl = pw, *pr = pw + m, *pidx = pw + 2 * m, *pidx2 = pw + 3 * m;
  k_join_fill<<<grid_for(nl), 256, 0, s>>>(d_lkey, nl, d_first, d_cnt, d_off, d_srow, pkey, pl, pr);
  k_iota<<<grid_for(m), 256, 0, s>>>(pidx, m);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, pkey, pkey + m, pidx, pidx2, (int)m, 0, 64, s);
  rc = with_temp(bytes, s, [&](void* t) {
    cub::DeviceRadixSort::SortPairs(t, bytes, pkey, pkey + m, pidx, pidx2, (int)m, 0, 64, s);
  });
  if (!rc) {
    k_take<<<grid_for(m), 256, 0, s>>>(pl, pidx2, m, d_left);
    k_take<<<grid_for(m), 256, 0, s>>>(pr, pidx2, m, d_right);
    rc = tcheck(cudaGetLastError(), "join order");
  }
  cudaFreeAsync(pkey, s);
  cudaFreeAsync(pw, s);
  return rc;
}

int fbx_first_repeat(const unsigned long long* d_skey, const unsigned* d_srow,
                     unsigned long long n_valid, unsigned long long* d_best, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = tcheck(cudaMemsetAsync(d_best, 0xFF, sizeof(ull), s), "repeat init");
  if (rc || n_valid < 2) return rc;
  k_first_repeat<<<grid_for(n_valid), 256, 0, s>>>(d_skey, d_srow, n_valid, d_best);
  return tcheck(cudaGetLastError(), "fbx_first_repeat");
}

int fbx_idset_entries(const unsigned long long* d_set, const unsigned long long* d_win_rows,
                      const unsigned long long* d_later_rows, unsigned long long cap,
                      unsigned long long* d_ids, unsigned long long* d_rows,
                      unsigned long long* d_count, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = tcheck(cudaMemsetAsync(d_count, 0, sizeof(ull), s), "entries count");
  if (rc) return rc;
  k_idset_entries<<<grid_for(cap + 1), 256, 0, s>>>(d_set, d_win_rows, d_later_rows, cap, d_ids,
                                                    d_rows, d_count);
  return tcheck(cudaGetLastError(), "fbx_idset_entries");
}

int fbx_seen_before(const unsigned long long* d_ids, const unsigned long long* d_rows,
                    unsigned long long n, const unsigned long long* d_prior,
                    unsigned long long n_prior, unsigned long long* d_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc = tcheck(cudaMemsetAsync(d_out, 0xFF, 2 * sizeof(ull), s), "seen init");
  if (rc || n == 0 || n_prior == 0) return rc;
  ull* sorted = nullptr;
  rc = tcheck(cudaMallocAsync((void**)&sorted, n_prior * sizeof(ull), s), "seen sort");
  if (rc) return rc;
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, d_prior, sorted, (int)n_prior, 0, 64, s);
  rc = with_temp(bytes, s, [&](void* t) {
    cub::DeviceRadixSort::SortKeys(t, bytes, d_prior, sorted, (int)n_prior, 0, 64, s);
  });
  if (!rc) {
    k_seen_before<<<grid_for(n), 256, 0, s>>>(d_ids, d_rows, n, sorted, n_prior, d_out);
    k_seen_before_id<<<grid_for(n), 256, 0, s>>>(d_ids, d_rows, n, d_out);
    rc = tcheck(cudaGetLastError(), "fbx_seen_before");
  }
  cudaFreeAsync(sorted, s);
  return rc;
}

}  // extern "C"
