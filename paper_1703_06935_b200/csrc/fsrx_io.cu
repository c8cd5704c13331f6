// FSRX decomposition files (format from the reference
// specification SPEC.md:248 -- the reference ships no implementation).
//
// Little-endian, in order:
//   "FSRX"  u32 version = 1  u64 n  u32 r  u8 variant  u64 seed  f64 alpha_hint
//   r x f64 eigenvalues
//   u8 storage (0 dense, 1 CSR) -- the spec's "U either dense or CSR" needs a tag
//   dense: n*r x f32 (row-major)
//   CSR:   u64 nnz, (n+1) x u64 row offsets, nnz x u32 columns, nnz x f32 values
//   n x f32 eta
//   u64 c, c x u64 component sizes, n x u64 permutation (block order)
//   u32 CRC-32 (IEEE 802.3, zlib's polynomial) of every preceding byte
//
// Host-side code: the caller moves U to/from the device around these calls.
#include <cstdio>
#include <cstring>
#include <vector>

#include "fsr_common.cuh"

namespace {

uint32_t crc_table[256];
bool crc_ready = false;

void crc_init() {
  if (crc_ready) return;
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    crc_table[i] = c;
  }
  crc_ready = true;
}

uint32_t crc_update(uint32_t crc, const void* data, size_t len) {
  const uint8_t* p = (const uint8_t*)data;
  crc = ~crc;
  for (size_t i = 0; i < len; ++i) crc = crc_table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
  return ~crc;
}

struct Writer {
  FILE* f;
  uint32_t crc = 0;
  bool ok = true;
  void put(const void* p, size_t bytes) {
    if (!ok || !bytes) return;
    ok = fwrite(p, 1, bytes, f) == bytes;
    crc = crc_update(crc, p, bytes);
  }
  template <typename T>
  void pod(T v) { put(&v, sizeof(T)); }
};

struct Reader {
  FILE* f;
  uint32_t crc = 0;
  bool ok = true;
  void get(void* p, size_t bytes) {
    if (!ok || !bytes) return;
    ok = fread(p, 1, bytes, f) == bytes;
    if (ok) crc = crc_update(crc, p, bytes);
  }
  template <typename T>
  T pod() {
    T v{};
    get(&v, sizeof(T));
    return v;
  }
};

constexpr uint32_t kVersion = 1;

}  // namespace

extern "C" {

int fsr_fsrx_write(fsr_ctx* ctx, const char* path, const fsr_fsrx_header* h, const double* eigenvalues,
                   const float* U_dense, const uint64_t* indptr, const uint32_t* indices, const float* values,
                   const float* eta, const uint64_t* sizes, const uint64_t* permutation) {
  FSR_REQUIRE(ctx, path && h && eigenvalues && eta && sizes && permutation, "fsrx_write: missing argument");
  FSR_REQUIRE(ctx, h->storage == 0 ? U_dense != nullptr : (indptr && (h->nnz == 0 || (indices && values))),
              "fsrx_write: missing U");
  crc_init();
  FILE* f = fopen(path, "wb");
  if (!f) return fsr::set_error(ctx, FSR_EIO, "fsrx_write: cannot open %s", path);
  Writer w{f};
  w.put("FSRX", 4);
  w.pod<uint32_t>(kVersion);
  w.pod<uint64_t>(h->n);
  w.pod<uint32_t>(h->r);
  w.pod<uint8_t>(h->variant);
  w.pod<uint64_t>(h->seed);
  w.pod<double>(h->alpha_hint);
  w.put(eigenvalues, sizeof(double) * h->r);
  w.pod<uint8_t>(h->storage);
  if (h->storage == 0) {
    w.put(U_dense, sizeof(float) * h->n * h->r);
  } else {
    w.pod<uint64_t>(h->nnz);
    w.put(indptr, sizeof(uint64_t) * (h->n + 1));
    w.put(indices, sizeof(uint32_t) * h->nnz);
    w.put(values, sizeof(float) * h->nnz);
  }
  w.put(eta, sizeof(float) * h->n);
  w.pod<uint64_t>(h->components);
  w.put(sizes, sizeof(uint64_t) * h->components);
  w.put(permutation, sizeof(uint64_t) * h->n);
  const uint32_t crc = w.crc;
  w.ok = w.ok && fwrite(&crc, 1, 4, f) == 4;
  const bool closed = fclose(f) == 0;
  if (!w.ok || !closed) return fsr::set_error(ctx, FSR_EIO, "fsrx_write: write to %s failed", path);
  return FSR_OK;
}

int fsr_fsrx_read_header(fsr_ctx* ctx, const char* path, fsr_fsrx_header* h) {
  FSR_REQUIRE(ctx, path && h, "fsrx_read_header: missing argument");
  FILE* f = fopen(path, "rb");
  if (!f) return fsr::set_error(ctx, FSR_EIO, "fsrx: cannot open %s", path);
  crc_init();
  Reader rd{f};
  char magic[4] = {0, 0, 0, 0};
  rd.get(magic, 4);
  const uint32_t version = rd.pod<uint32_t>();
  memset(h, 0, sizeof(*h));
  h->n = rd.pod<uint64_t>();
  h->r = rd.pod<uint32_t>();
  h->variant = rd.pod<uint8_t>();
  h->seed = rd.pod<uint64_t>();
  h->alpha_hint = rd.pod<double>();
  bool ok = rd.ok && !memcmp(magic, "FSRX", 4) && version == kVersion;
  if (ok && fseek(f, (long)(sizeof(double) * h->r), SEEK_CUR) == 0) {
    rd.get(&h->storage, 1);
    if (h->storage == 1) h->nnz = rd.pod<uint64_t>();
    ok = rd.ok && h->storage <= 1;
  } else {
    ok = false;
  }
  if (ok) {
    const long skip = h->storage == 0 ? (long)(sizeof(float) * h->n * h->r)
                                      : (long)(sizeof(uint64_t) * (h->n + 1) + (sizeof(uint32_t) + sizeof(float)) * h->nnz);
    ok = fseek(f, skip + (long)(sizeof(float) * h->n), SEEK_CUR) == 0;
    if (ok) {
      h->components = rd.pod<uint64_t>();
      ok = rd.ok;
    }
  }
  fclose(f);
  if (!ok) return fsr::set_error(ctx, FSR_EIO, "fsrx: %s is not a version-1 FSRX file", path);
  return FSR_OK;
}

int fsr_fsrx_read(fsr_ctx* ctx, const char* path, fsr_fsrx_header* h, double* eigenvalues, float* U_dense,
                  uint64_t* indptr, uint32_t* indices, float* values, float* eta, uint64_t* sizes,
                  uint64_t* permutation) {
  FSR_REQUIRE(ctx, path && h && eigenvalues && eta && sizes && permutation, "fsrx_read: missing argument");
  fsr_fsrx_header want;
  FSR_TRY(fsr_fsrx_read_header(ctx, path, &want));
  FSR_REQUIRE(ctx, want.storage == 0 ? U_dense != nullptr : (indptr && (want.nnz == 0 || (indices && values))),
              "fsrx_read: missing U buffers");
  FILE* f = fopen(path, "rb");
  if (!f) return fsr::set_error(ctx, FSR_EIO, "fsrx: cannot open %s", path);
  Reader rd{f};
  char magic[4];
  rd.get(magic, 4);
  rd.pod<uint32_t>();
  *h = want;
  rd.pod<uint64_t>();
  rd.pod<uint32_t>();
  rd.pod<uint8_t>();
  rd.pod<uint64_t>();
  rd.pod<double>();
  rd.get(eigenvalues, sizeof(double) * h->r);
  rd.pod<uint8_t>();
  if (h->storage == 0) {
    rd.get(U_dense, sizeof(float) * h->n * h->r);
  } else {
    rd.pod<uint64_t>();
    rd.get(indptr, sizeof(uint64_t) * (h->n + 1));
    rd.get(indices, sizeof(uint32_t) * h->nnz);
    rd.get(values, sizeof(float) * h->nnz);
  }
  rd.get(eta, sizeof(float) * h->n);
  rd.pod<uint64_t>();
  rd.get(sizes, sizeof(uint64_t) * h->components);
  rd.get(permutation, sizeof(uint64_t) * h->n);
  const uint32_t computed = rd.crc;
  uint32_t stored = 0;
  const bool got = fread(&stored, 1, 4, f) == 4;
  char extra;
  const bool at_end = fread(&extra, 1, 1, f) == 0;
  fclose(f);
  if (!rd.ok || !got) return fsr::set_error(ctx, FSR_EIO, "fsrx: %s is truncated", path);
  if (stored != computed || !at_end)
    return fsr::set_error(ctx, FSR_EIO, "fsrx: checksum mismatch in %s (stored %08x, computed %08x)", path, stored,
                          computed);
  return FSR_OK;
}

}  // extern "C"
