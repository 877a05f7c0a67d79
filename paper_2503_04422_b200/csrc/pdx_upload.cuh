// Block-record upload shared by the .pdx loader and pdx_index_create: block
// images [d][m_padded] (the reference's Block.data) stream through pinned
// staging into the store's tile layout; the GPU transposes chunk i while the
// host produces chunk i+1.
#pragma once
#include <vector>

#include "pdx_common.cuh"

namespace pdx {
namespace {

constexpr int64_t kChunkBytes = 64ll << 20;
constexpr int64_t kChunkTiles = 1 << 16;

// One 64-slot tile of a block image in the staging buffer.
struct TileSrc {
  int64_t raw_off;  // float offset of the block image [d][mp] in staging
  int64_t tile;     // destination tile in the store
  int32_t mp;       // the block's m_padded (image row length)
  int32_t col;      // first block column of this tile (64 * tile-in-block)
  int32_t valid;    // block columns of this tile that hold vectors
  int32_t _pad;
};

// file image [d][mp] -> tile [d_pad/G][64][G]; dims >= d and slots >= valid are 0
__global__ void __launch_bounds__(256) blocks_to_tiles_kernel(const float* __restrict__ raw,
                                                              const TileSrc* __restrict__ src,
                                                              int d, int d_pad, int group,
                                                              float* __restrict__ tiles) {
  const TileSrc s = src[blockIdx.x];
  float* out = tiles + s.tile * (int64_t)d_pad * kTile;
  const int total = d_pad * kTile;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int j, i;
    if (group == 8) {
      const int r = e & 511;
      j = (e >> 9) * 8 + (r & 7);
      i = r >> 3;
    } else {
      j = e >> 6;
      i = e & 63;
    }
    float v = 0.f;
    if (j < d && i < s.valid) v = raw[s.raw_off + (int64_t)j * s.mp + s.col + i];
    out[e] = v;
  }
}

// tile -> file image columns [col, col + valid) of every dim row
__global__ void __launch_bounds__(256) tiles_to_blocks_kernel(const float* __restrict__ tiles,
                                                              const TileSrc* __restrict__ src,
                                                              int d, int d_pad, int group,
                                                              float* __restrict__ raw) {
  const TileSrc s = src[blockIdx.x];
  const float* in = tiles + s.tile * (int64_t)d_pad * kTile;
  const int total = d * kTile;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int j = e >> 6, i = e & 63;
    if (i >= s.valid) continue;
    const float v = group == 8 ? in[((j >> 3) * kTile + i) * 8 + (j & 7)] : in[j * kTile + i];
    raw[s.raw_off + (int64_t)j * s.mp + s.col + i] = v;
  }
}

// RAII for the staging resources of one transfer
struct Staging {
  float* h_raw[2] = {nullptr, nullptr};
  float* d_raw[2] = {nullptr, nullptr};
  TileSrc* d_src[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Staging() {
    for (int b = 0; b < 2; ++b) {
      if (ev[b]) cudaEventSynchronize(ev[b]), cudaEventDestroy(ev[b]);
      if (h_raw[b]) cudaFreeHost(h_raw[b]);
      if (d_raw[b]) cudaFree(d_raw[b]);
      if (d_src[b]) cudaFree(d_src[b]);
    }
  }
  int alloc(int64_t bytes, int nbuf) {
    for (int b = 0; b < nbuf; ++b) {
      PDX_CUDA_CHECK(cudaMallocHost(&h_raw[b], (size_t)bytes));
      PDX_CUDA_CHECK(cudaMalloc(&d_raw[b], (size_t)bytes));
      PDX_CUDA_CHECK(cudaMalloc(&d_src[b], sizeof(TileSrc) * kChunkTiles));
      PDX_CUDA_CHECK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    return PDX_OK;
  }
};


// Streams nblocks block records into tiles.  `src` supplies them in order:
//   int head(int64_t b, uint32_t mm[2])       -> m, m_padded of block b
//   int body(int64_t b, int64_t m, int64_t floats, int64_t* ids, float* data)
// (data: the [d][m_padded] image).  Fills h_block_m / h_block_mpad.
template <class Src>
int upload_blocks(Src& src, int64_t nblocks, int64_t d, int group, int64_t max_block_bytes,
                  float* d_tiles, int64_t* d_tile_ids, int32_t* h_block_m,
                  int32_t* h_block_mpad, cudaStream_t st) {
  const int d_pad = group == 8 ? (int)((d + 7) / 8 * 8) : (int)d;
  const int64_t cap = max_block_bytes > kChunkBytes ? max_block_bytes : kChunkBytes;
  Staging S;
  PDX_TRY(S.alloc(cap, 2));
  std::vector<TileSrc> tsrc[2];
  std::vector<int64_t> ids[2];
  std::vector<int64_t> bids;
  int cur = 0;
  int64_t used = 0, tile = 0, chunk_tile0 = 0;
  auto flush = [&]() -> int {
    const int64_t nt = (int64_t)tsrc[cur].size();
    if (nt > 0) {
      PDX_CUDA_CHECK(cudaMemcpyAsync(S.d_raw[cur], S.h_raw[cur], (size_t)used * 4,
                                     cudaMemcpyHostToDevice, st));
      PDX_CUDA_CHECK(cudaMemcpyAsync(S.d_src[cur], tsrc[cur].data(), sizeof(TileSrc) * nt,
                                     cudaMemcpyHostToDevice, st));
      PDX_CUDA_CHECK(cudaMemcpyAsync(d_tile_ids + chunk_tile0 * kTile, ids[cur].data(),
                                     sizeof(int64_t) * kTile * nt, cudaMemcpyHostToDevice, st));
      blocks_to_tiles_kernel<<<(unsigned)nt, 256, 0, st>>>(S.d_raw[cur], S.d_src[cur], (int)d,
                                                           d_pad, group, d_tiles);
      PDX_LAUNCH_CHECK();
    }
    PDX_CUDA_CHECK(cudaEventRecord(S.ev[cur], st));
    cur ^= 1;
    PDX_CUDA_CHECK(cudaEventSynchronize(S.ev[cur]));  // the other buffer is free again
    tsrc[cur].clear();
    ids[cur].clear();
    used = 0;
    chunk_tile0 = tile;
    return PDX_OK;
  };
  for (int64_t b = 0; b < nblocks; ++b) {
    uint32_t mm[2];
    PDX_TRY(src.head(b, mm));
    const int64_t m = mm[0], mp = mm[1], floats = d * mp;
    const int64_t nt = (m + kTile - 1) / kTile;
    PDX_REQUIRE(mp >= m, "block %lld: m_padded %lld < m %lld", (long long)b, (long long)mp,
                (long long)m);
    PDX_REQUIRE(nt <= kChunkTiles, "block %lld spans more than %lld tiles", (long long)b,
                (long long)kChunkTiles);
    if (used + floats > cap / 4 || (int64_t)tsrc[cur].size() + nt > kChunkTiles) PDX_TRY(flush());
    h_block_m[b] = (int32_t)m;
    h_block_mpad[b] = (int32_t)mp;
    bids.resize((size_t)m);
    PDX_TRY(src.body(b, m, floats, bids.data(), S.h_raw[cur] + used));
    for (int64_t u = 0; u < nt; ++u) {
      const int32_t valid = (int32_t)(m - u * kTile < kTile ? m - u * kTile : kTile);
      tsrc[cur].push_back(TileSrc{used, tile, (int32_t)mp, (int32_t)(u * kTile), valid, 0});
      for (int i = 0; i < kTile; ++i) ids[cur].push_back(i < valid ? bids[u * kTile + i] : -1);
      ++tile;
    }
    used += floats;
  }
  PDX_TRY(flush());
  PDX_CUDA_CHECK(cudaStreamSynchronize(st));
  return PDX_OK;
}

}  // namespace
}  // namespace pdx
