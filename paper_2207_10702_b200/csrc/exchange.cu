// exchange.cu — a6 in the large-|M| regime: the touched-set dM exchange.
//
// A linear's tiles sit at static offsets, so the only slots of dM it can ever write are the
// union of [off_t, off_t + Z1 Z2) over its tiles; an embedding writes chunks of its own
// memory (all of M under GMS, its segment under LMS, or — for small tables such as a bias
// via L — exactly the chunks of its rows).  Every other slot of dM stays zero on every rank,
// so summing it over ranks moves |M| - |touched| zeros across NVLink.  When |M| exceeds the
// virtual model (C5: |M| up to 512 M elements for a 16.8 M-element layer) the exchange
// packs the touched intervals into one contiguous buffer, all-reduces that, and unpacks it:
// NVLink traffic <= min(|M|, n) elements instead of |M|.
//
// Intervals are computed on the host once per module set (sorted, merged); pack / unpack
// are HBM-bound gathers / scatters of 16-byte vectors (interval bounds are multiples of
// A = 8 elements whenever A % 4 == 0, so no vector straddles two intervals).
#include <algorithm>
#include <type_traits>
#include <vector>

#include "roast_internal.h"

namespace roast {
namespace {

// dir 0: buf[p] = dM[start_i + p - prefix_i];  dir 1: dM[...] = scale * buf[p]
template <int V>
__global__ void pack_kernel(float* __restrict__ dM, float* __restrict__ buf, const int64_t* __restrict__ start,
                            const int64_t* __restrict__ prefix, int n_iv, int64_t total, int dir, float scale) {
  using VT = typename std::conditional<V == 4, float4, float>::type;
  int64_t b, e;
  cta_range(total, V, &b, &e);
  IvWalk w{start, prefix, n_iv};
  if (b + int64_t(threadIdx.x) * V < e) w.seek(b + int64_t(threadIdx.x) * V);
  for (int64_t p = b + int64_t(threadIdx.x) * V; p < e; p += int64_t(blockDim.x) * V) {
    const int64_t src = w.slot(p);
    VT* d = reinterpret_cast<VT*>(dM + src);
    VT* bp = reinterpret_cast<VT*>(buf + p);
    if (dir == 0) {
      *bp = *d;
    } else {
      VT v = *bp;
      if constexpr (V == 4) {
        v.x *= scale; v.y *= scale; v.z *= scale; v.w *= scale;
      } else {
        v *= scale;
      }
      *d = v;
    }
  }
}

}  // namespace

// Sort + merge [s_i, s_i + span) (span > 0) into disjoint, non-adjacent intervals.
void merge_intervals(std::vector<std::pair<int64_t, int64_t>>& iv) {
  std::sort(iv.begin(), iv.end());
  size_t w = 0;
  for (size_t r = 0; r < iv.size(); ++r) {
    if (w > 0 && iv[r].first <= iv[w - 1].second)
      iv[w - 1].second = std::max(iv[w - 1].second, iv[r].second);
    else
      iv[w++] = iv[r];
  }
  iv.resize(w);
}

// The touched set of the registered modules (see the header comment); rebuilt when modules change.
roast_status_t touched_prepare(Ctx* c, cudaStream_t s) {
  if (c->touched_for == int64_t(c->modules.size()) && c->touched_valid) return ROAST_OK;
  std::vector<std::pair<int64_t, int64_t>> iv;
  const int64_t span = int64_t(c->tile.z1) * c->tile.z2;
  for (const Module& m : c->modules) {
    if (m.kind == kLinear) {
      for (int64_t off : m.h_off) iv.emplace_back(off, off + span);
    } else {
      const int64_t nchunks = m.rows * m.chunks_per_row;
      if (nchunks <= (int64_t(1) << 16)) {   // small table (e.g. a bias via L): its exact chunks
        for (int64_t k = 0; k < nchunks; ++k) {
          const int64_t off = int64_t(m.hash.offset(uint64_t(k)));
          iv.emplace_back(off, off + m.chunk);
        }
      } else {   // every legal chunk position of its memory
        const int64_t b = int64_t(m.hash.base);
        iv.emplace_back(b, b + int64_t(m.hash.align) * int64_t(m.hash.R - 1) + m.chunk);
      }
    }
  }
  merge_intervals(iv);
  int64_t total = 0;
  bool vec = true;
  std::vector<int64_t> host(2 * iv.size() + 1);
  for (size_t i = 0; i < iv.size(); ++i) {
    host[i] = iv[i].first;
    host[iv.size() + i] = total;
    total += iv[i].second - iv[i].first;
    vec = vec && iv[i].first % 4 == 0 && (iv[i].second - iv[i].first) % 4 == 0;
  }
  host[2 * iv.size()] = total;
  cudaFree(c->d_iv);
  cudaFree(c->d_pack);
  c->d_iv = nullptr;
  c->d_pack = nullptr;
  c->touched_valid = false;
  if (!iv.empty()) {
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->d_iv), host.size() * sizeof(int64_t)));
    ROAST_CUDA_CHECK(cudaMemcpy(c->d_iv, host.data(), host.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->d_pack), size_t(total) * sizeof(float)));
  }
  c->n_iv = int32_t(iv.size());
  c->touched_n = total;
  c->touched_vec = vec;
  c->touched_for = int64_t(c->modules.size());
  c->touched_valid = true;
  (void)s;
  return ROAST_OK;
}

cudaError_t launch_pack(Ctx* c, int dir, float scale, cudaStream_t s) {
  if (c->touched_n == 0) return cudaSuccess;
  const int64_t* start = c->d_iv;
  const int64_t* prefix = c->d_iv + c->n_iv;
  const int V = c->touched_vec ? 4 : 1;
  int64_t blocks = (c->touched_n / V + 255) / 256;
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 8);
  if (V == 4)
    pack_kernel<4><<<unsigned(blocks), 256, 0, s>>>(c->dM, c->d_pack, start, prefix, c->n_iv, c->touched_n, dir, scale);
  else
    pack_kernel<1><<<unsigned(blocks), 256, 0, s>>>(c->dM, c->d_pack, start, prefix, c->n_iv, c->touched_n, dir, scale);
  return cudaGetLastError();
}

}  // namespace roast

using namespace roast;

extern "C" {

roast_status_t roast_touched_intervals(const int64_t* starts_in, int64_t n, int64_t span, int64_t* starts_out,
                                       int64_t* lens_out, int64_t cap, int64_t* count) {
  if ((n > 0 && !starts_in) || !count || span <= 0 || n < 0 || cap < 0) return fail(ROAST_ERR_CONFIG, "bad arguments");
  std::vector<std::pair<int64_t, int64_t>> iv;
  iv.reserve(size_t(n));
  for (int64_t i = 0; i < n; ++i) iv.emplace_back(starts_in[i], starts_in[i] + span);
  merge_intervals(iv);
  *count = int64_t(iv.size());
  if (*count > cap) return fail(ROAST_ERR_CAPACITY, "more intervals than cap");
  if (*count && (!starts_out || !lens_out)) return fail(ROAST_ERR_CONFIG, "null output");
  for (size_t i = 0; i < iv.size(); ++i) {
    starts_out[i] = iv[i].first;
    lens_out[i] = iv[i].second - iv[i].first;
  }
  return ROAST_OK;
}

roast_status_t roast_set_exchange(roast_t h, int32_t mode) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (mode < ROAST_EXCHANGE_AUTO || mode > ROAST_EXCHANGE_TOUCHED) return fail(ROAST_ERR_CONFIG, "bad exchange mode");
  c->exchange_mode = mode;
  return ROAST_OK;
}

roast_status_t roast_touched_size(roast_t h, int64_t* n_touched, int64_t* n_intervals) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (roast_status_t st = touched_prepare(c, 0)) return st;
  if (n_touched) *n_touched = c->touched_n;
  if (n_intervals) *n_intervals = c->n_iv;
  return ROAST_OK;
}

roast_status_t roast_debug_exchange(roast_t h, float scale, roast_stream_t stream) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (roast_status_t st = touched_prepare(c, s)) return st;
  ROAST_CUDA_CHECK(launch_pack(c, 0, 1.f, s));
  ROAST_CUDA_CHECK(launch_pack(c, 1, scale, s));
  c->launches += 2;
  return ROAST_OK;
}

}  // extern "C"
