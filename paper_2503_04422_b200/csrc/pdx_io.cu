// .pdx store interchange, HBM <-> file (storage.py:115-194 of the reference).
//
// The reference reads the whole file into host memory and builds a list of
// numpy Blocks.  Here the block records stream through two pinned staging
// buffers: while the GPU transposes chunk i from the file's dimension-major
// block images [d][m_padded] into the store's tile layout (K1's output
// format), the host reads chunk i+1.  Saving runs the inverse transposition
// chunk by chunk and writes byte-identical records.
#include <sys/stat.h>

#include <cerrno>
#include <vector>

#include "pdx_common.cuh"
#include "pdx_upload.cuh"

namespace pdx {

namespace {

constexpr char kMagic[8] = {'P', 'D', 'X', 'v', '1', 0, 0, 0};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kFlagTransform = 1, kFlagIvf = 2;
constexpr int64_t kHeaderBytes = 40;  // struct "<8sIIQIIII"

#define PDX_FORMAT(...)              \
  do {                               \
    ::pdx::set_error(__VA_ARGS__);   \
    return PDX_EFORMAT;              \
  } while (0)

struct File {
  FILE* f = nullptr;
  const char* path;
  int64_t size = 0;
  int64_t pos = 0;
  std::vector<char> vbuf;
  explicit File(const char* p) : path(p) {}
  ~File() {
    if (f) fclose(f);
  }
};

int open_read(File& F) {
  F.f = fopen(F.path, "rb");
  if (!F.f) {
    set_error("%s: %s", F.path, strerror(errno));
    return PDX_EIO;
  }
  struct stat st;
  if (fstat(fileno(F.f), &st) != 0) {
    set_error("%s: %s", F.path, strerror(errno));
    return PDX_EIO;
  }
  F.size = (int64_t)st.st_size;
  F.vbuf.resize(8 << 20);
  setvbuf(F.f, F.vbuf.data(), _IOFBF, F.vbuf.size());
  return PDX_OK;
}

// read exactly n bytes (dst may be null: skip)
int take(File& F, void* dst, int64_t n) {
  if (n < 0 || F.pos + n > F.size) PDX_FORMAT("%s: truncated at byte offset %lld", F.path, (long long)F.pos);
  if (dst) {
    if ((int64_t)fread(dst, 1, (size_t)n, F.f) != n) {
      set_error("%s: read failed at byte offset %lld", F.path, (long long)F.pos);
      return PDX_EIO;
    }
  } else if (n && fseeko(F.f, (off_t)(F.pos + n), SEEK_SET) != 0) {
    set_error("%s: seek failed at byte offset %lld", F.path, (long long)F.pos);
    return PDX_EIO;
  }
  F.pos += n;
  return PDX_OK;
}


int read_header(File& F, pdx_file_info* I) {
  unsigned char h[kHeaderBytes];
  PDX_TRY(take(F, h, kHeaderBytes));
  if (memcmp(h, kMagic, 8) != 0) PDX_FORMAT("%s: bad magic", F.path);
  uint32_t version, flags, d, bs, bc, reserved;
  uint64_t n;
  memcpy(&version, h + 8, 4);
  memcpy(&flags, h + 12, 4);
  memcpy(&n, h + 16, 8);
  memcpy(&d, h + 24, 4);
  memcpy(&bs, h + 28, 4);
  memcpy(&bc, h + 32, 4);
  memcpy(&reserved, h + 36, 4);
  if (version != kVersion) PDX_FORMAT("%s: unsupported version %u", F.path, version);
  if (d < 1 || d > 65535) PDX_FORMAT("%s: dimensionality %u unsupported", F.path, d);
  memset(I, 0, sizeof(*I));
  I->n = (int64_t)n;
  I->d = (int32_t)d;
  I->block_size = (int32_t)bs;
  I->nblocks = bc;
  I->flags = (int32_t)flags;
  return PDX_OK;
}

struct Layout {
  int64_t means_at, transform_at, blocks_at, ivf_at;
};

// Walk the sections; fills the info's counts and the section offsets.
int walk(File& F, pdx_file_info* I, Layout* L) {
  PDX_TRY(read_header(F, I));
  const int64_t d = I->d;
  L->means_at = F.pos;
  PDX_TRY(take(F, nullptr, 8 * d));
  L->transform_at = F.pos;
  if (I->flags & kFlagTransform) {
    PDX_TRY(take(F, &I->transform_seed, 8));
    PDX_TRY(take(F, nullptr, 4 * d * d));
  }
  L->blocks_at = F.pos;
  int64_t total = 0;
  for (int64_t b = 0; b < I->nblocks; ++b) {
    uint32_t mm[2];
    PDX_TRY(take(F, mm, 8));
    if (mm[1] < mm[0]) PDX_FORMAT("%s: block %lld has m_padded %u < m %u", F.path, (long long)b, mm[1], mm[0]);
    const int64_t bytes = 4 * d * (int64_t)mm[1];
    PDX_TRY(take(F, nullptr, 8 * (int64_t)mm[0] + bytes));
    total += mm[0];
    I->ntiles += (mm[0] + kTile - 1) / kTile;
    if (bytes > I->max_block_bytes) I->max_block_bytes = bytes;
  }
  L->ivf_at = F.pos;
  if (I->flags & kFlagIvf) {
    unsigned char h[12];
    PDX_TRY(take(F, h, 12));
    uint32_t nlist;
    memcpy(&nlist, h, 4);
    memcpy(&I->training_seed, h + 4, 8);
    if (nlist < 1 || nlist > 0x7fffffffu) PDX_FORMAT("%s: bad nlist %u", F.path, nlist);
    I->nlist = (int32_t)nlist;
    PDX_TRY(take(F, nullptr, 4 * (int64_t)nlist * d + 4 * ((int64_t)nlist + 1) +
                                 8 * (int64_t)nlist * d));
  }
  if (total != I->n)
    PDX_FORMAT("%s: header claims %lld vectors, blocks hold %lld", F.path, (long long)I->n,
               (long long)total);
  return PDX_OK;
}

}  // namespace
}  // namespace pdx

using namespace pdx;

extern "C" int pdx_file_probe(const char* path, pdx_file_info* info) {
  PDX_REQUIRE(path && info, "pdx_file_probe: null argument");
  File F(path);
  PDX_TRY(open_read(F));
  Layout L;
  return walk(F, info, &L);
}

extern "C" int pdx_file_load(const char* path, const pdx_file_info* info, int32_t group,
                             float* d_tiles, int64_t* d_tile_ids, int32_t* h_block_m,
                             int32_t* h_block_mpad, double* h_global_means, float* h_transform,
                             float* h_centroids, int64_t* h_bucket_offsets,
                             double* h_bucket_means, void* stream) {
  PDX_REQUIRE(path && info, "pdx_file_load: null argument");
  PDX_REQUIRE(group == 1 || group == 8, "group must be 1 or 8");
  File F(path);
  PDX_TRY(open_read(F));
  pdx_file_info I;
  Layout L;
  PDX_TRY(walk(F, &I, &L));
  PDX_REQUIRE(I.n == info->n && I.nblocks == info->nblocks && I.ntiles == info->ntiles &&
                  I.d == info->d,
              "%s changed since it was probed", path);
  PDX_REQUIRE(I.ntiles == 0 || (d_tiles && d_tile_ids), "pdx_file_load: null tile buffers");
  PDX_REQUIRE(I.nblocks == 0 || (h_block_m && h_block_mpad), "pdx_file_load: null block arrays");
  PDX_REQUIRE(!(I.flags & kFlagTransform) || h_transform, "pdx_file_load: file has a rotation");
  PDX_REQUIRE(!(I.flags & kFlagIvf) || (h_centroids && h_bucket_offsets && h_bucket_means),
              "pdx_file_load: file has an IVF section");
  const int64_t d = I.d;
  cudaStream_t st = as_stream(stream);

  if (fseeko(F.f, (off_t)L.means_at, SEEK_SET) != 0) {
    set_error("%s: seek failed", path);
    return PDX_EIO;
  }
  F.pos = L.means_at;
  std::vector<double> means(d);
  PDX_TRY(take(F, means.data(), 8 * d));
  if (h_global_means) memcpy(h_global_means, means.data(), 8 * d);
  if (I.flags & kFlagTransform) {
    PDX_TRY(take(F, nullptr, 8));
    PDX_TRY(take(F, h_transform, 4 * d * d));
  }

  struct FileSrc {
    File& F;
    int head(int64_t, uint32_t* mm) { return take(F, mm, 8); }
    int body(int64_t, int64_t m, int64_t floats, int64_t* ids, float* data) {
      PDX_TRY(take(F, ids, 8 * m));
      return take(F, data, 4 * floats);
    }
  } src{F};
  PDX_TRY(upload_blocks(src, I.nblocks, d, group, I.max_block_bytes, d_tiles, d_tile_ids,
                        h_block_m, h_block_mpad, st));
  if (I.flags & kFlagIvf) {
    PDX_TRY(take(F, nullptr, 12));
    PDX_TRY(take(F, h_centroids, 4 * (int64_t)I.nlist * d));
    std::vector<uint32_t> off((size_t)I.nlist + 1);
    PDX_TRY(take(F, off.data(), 4 * ((int64_t)I.nlist + 1)));
    for (int64_t c = 0; c <= I.nlist; ++c) h_bucket_offsets[c] = off[c];
    PDX_TRY(take(F, h_bucket_means, 8 * (int64_t)I.nlist * d));
  }
  PDX_CUDA_CHECK(cudaStreamSynchronize(st));
  return PDX_OK;
}

namespace {
int put(FILE* f, const char* path, const void* p, int64_t n) {
  if (n && (int64_t)fwrite(p, 1, (size_t)n, f) != n) {
    set_error("%s: %s", path, strerror(errno));
    return PDX_EIO;
  }
  return PDX_OK;
}
}  // namespace

extern "C" int pdx_file_save(const char* path, const pdx_store* store, int32_t block_size,
                             const int32_t* h_block_mpad, const double* h_global_means,
                             const float* h_transform, uint64_t transform_seed, int32_t nlist,
                             uint64_t training_seed, const float* h_centroids,
                             const int64_t* h_bucket_offsets, const double* h_bucket_means,
                             void* stream) {
  PDX_REQUIRE(path && store && h_global_means, "pdx_file_save: null argument");
  PDX_REQUIRE(nlist >= 0, "bad nlist");
  PDX_REQUIRE(nlist == 0 || (h_centroids && h_bucket_offsets && h_bucket_means),
              "pdx_file_save: IVF arrays required");
  PDX_REQUIRE(store->nblocks <= 0xffffffffll, "too many blocks for the .pdx format");
  const int64_t d = store->d, nb = store->nblocks;
  cudaStream_t st = as_stream(stream);
  std::vector<int64_t> btile((size_t)nb + 1, 0);
  std::vector<int32_t> bm((size_t)nb);
  if (nb) {
    PDX_CUDA_CHECK(cudaMemcpyAsync(btile.data(), store->d_block_tile, 8 * (nb + 1),
                                   cudaMemcpyDeviceToHost, st));
    PDX_CUDA_CHECK(cudaMemcpyAsync(bm.data(), store->d_block_m, 4 * nb, cudaMemcpyDeviceToHost, st));
    PDX_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  int64_t n = 0, maxb = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t mp = h_block_mpad ? h_block_mpad[b] : bm[b];
    PDX_REQUIRE(mp >= bm[b], "block %lld: m_padded %lld < m %d", (long long)b, (long long)mp, bm[b]);
    PDX_REQUIRE(btile[b + 1] - btile[b] == (bm[b] + kTile - 1) / kTile, "block %lld: tile count",
                (long long)b);
    n += bm[b];
    if (4 * d * mp > maxb) maxb = 4 * d * mp;
  }
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_error("%s: %s", path, strerror(errno));
    return PDX_EIO;
  }
  struct Closer {
    FILE* f;
    ~Closer() { if (f) fclose(f); }
  } closer{f};
  std::vector<char> vbuf(8 << 20);
  setvbuf(f, vbuf.data(), _IOFBF, vbuf.size());
  unsigned char h[kHeaderBytes];
  const uint32_t flags = (h_transform ? kFlagTransform : 0) | (nlist ? kFlagIvf : 0);
  const uint32_t ud = (uint32_t)d, ubs = (uint32_t)block_size, ubc = (uint32_t)nb, zero = 0;
  const uint64_t un = (uint64_t)n;
  memcpy(h, kMagic, 8);
  memcpy(h + 8, &kVersion, 4);
  memcpy(h + 12, &flags, 4);
  memcpy(h + 16, &un, 8);
  memcpy(h + 24, &ud, 4);
  memcpy(h + 28, &ubs, 4);
  memcpy(h + 32, &ubc, 4);
  memcpy(h + 36, &zero, 4);
  PDX_TRY(put(f, path, h, kHeaderBytes));
  PDX_TRY(put(f, path, h_global_means, 8 * d));
  if (h_transform) {
    PDX_TRY(put(f, path, &transform_seed, 8));
    PDX_TRY(put(f, path, h_transform, 4 * d * d));
  }
  const int64_t cap = maxb > kChunkBytes ? maxb : kChunkBytes;
  Staging S;
  PDX_TRY(S.alloc(cap, 1));
  std::vector<TileSrc> src;
  std::vector<int64_t> ids;
  int64_t b = 0;
  while (b < nb) {
    // a chunk of whole blocks
    int64_t e = b, used = 0;
    src.clear();
    while (e < nb) {
      const int64_t mp = h_block_mpad ? h_block_mpad[e] : bm[e];
      const int64_t nt = btile[e + 1] - btile[e];
      if (e > b && (used + d * mp > cap / 4 || (int64_t)src.size() + nt > kChunkTiles)) break;
      PDX_REQUIRE(nt <= kChunkTiles, "block %lld spans too many tiles", (long long)e);
      for (int64_t u = 0; u < nt; ++u) {
        const int32_t valid = (int32_t)(bm[e] - u * kTile < kTile ? bm[e] - u * kTile : kTile);
        src.push_back(TileSrc{used, btile[e] + u, (int32_t)mp, (int32_t)(u * kTile), valid, 0});
      }
      used += d * mp;
      ++e;
    }
    const int64_t t0 = btile[b], nt = btile[e] - btile[b];
    ids.resize((size_t)nt * kTile);
    if (used) PDX_CUDA_CHECK(cudaMemsetAsync(S.d_raw[0], 0, (size_t)used * 4, st));
    if (nt) {
      PDX_CUDA_CHECK(cudaMemcpyAsync(S.d_src[0], src.data(), sizeof(TileSrc) * nt,
                                     cudaMemcpyHostToDevice, st));
      tiles_to_blocks_kernel<<<(unsigned)nt, 256, 0, st>>>(store->d_tiles, S.d_src[0], (int)d,
                                                           store->d_pad, store->group, S.d_raw[0]);
      PDX_LAUNCH_CHECK();
      PDX_CUDA_CHECK(cudaMemcpyAsync(ids.data(), store->d_tile_ids + t0 * kTile,
                                     sizeof(int64_t) * kTile * nt, cudaMemcpyDeviceToHost, st));
    }
    if (used)
      PDX_CUDA_CHECK(cudaMemcpyAsync(S.h_raw[0], S.d_raw[0], (size_t)used * 4,
                                     cudaMemcpyDeviceToHost, st));
    PDX_CUDA_CHECK(cudaStreamSynchronize(st));
    int64_t off = 0;
    for (int64_t x = b; x < e; ++x) {
      const uint32_t mm[2] = {(uint32_t)bm[x], (uint32_t)(h_block_mpad ? h_block_mpad[x] : bm[x])};
      PDX_TRY(put(f, path, mm, 8));
      PDX_TRY(put(f, path, ids.data() + (btile[x] - t0) * kTile, 8 * (int64_t)bm[x]));
      PDX_TRY(put(f, path, S.h_raw[0] + off, 4 * d * mm[1]));
      off += d * mm[1];
    }
    b = e;
  }
  if (nlist) {
    const uint32_t unl = (uint32_t)nlist;
    PDX_TRY(put(f, path, &unl, 4));
    PDX_TRY(put(f, path, &training_seed, 8));
    PDX_TRY(put(f, path, h_centroids, 4 * (int64_t)nlist * d));
    std::vector<uint32_t> off((size_t)nlist + 1);
    for (int64_t c = 0; c <= nlist; ++c) {
      PDX_REQUIRE(h_bucket_offsets[c] >= 0 && h_bucket_offsets[c] <= nb, "bad bucket offset");
      off[c] = (uint32_t)h_bucket_offsets[c];
    }
    PDX_TRY(put(f, path, off.data(), 4 * ((int64_t)nlist + 1)));
    PDX_TRY(put(f, path, h_bucket_means, 8 * (int64_t)nlist * d));
  }
  if (fflush(f) != 0) {
    set_error("%s: %s", path, strerror(errno));
    return PDX_EIO;
  }
  return PDX_OK;
}
