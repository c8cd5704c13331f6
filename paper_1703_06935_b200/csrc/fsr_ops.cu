// Operator-level entry points: the reference's offline functions as single C
// calls, so a C/C++/Go/Java host gets range_finder /
// approx_eigendecomposition / decompose / sparsify without re-implementing
// the schedule the Python package used to own.  Host-side orchestration only:
// every numeric step is one of the primitives in this library (K0-K7), the
// device temporaries are stream-ordered (cudaMallocAsync on the context
// stream), and the schedule is the one spectral.py documents:
//
//   range_finder (reference spectral.py:147-171): K0 start block from
//     numpy's SeedSequence/Philox stream; q rounds of {orthonormalise, K2}.
//     fp32 fast mode (FSR_SI_SPAN_ONLY): rounds 1..q-1 only precondition
//     (span(Q) is what reaches the output); FSR_SI_FUSED_RR: the last round
//     is preconditioned and its exact Gram handed to Rayleigh-Ritz.
//   orthonormalise (spectral.py:165-169): CholeskyQR2 (first pass on a
//     7-bit Gram), Householder when Cholesky breaks down or the result misses
//     the re-orthogonalisation tolerance.
//   Rayleigh-Ritz (spectral.py:174-198): C = Q^T B, eigh (generalised with
//     G when given), U = Q V, column sign rule, eta.
//   sparsify (spectral.py:269-294): radix select of the tau-th |u| key,
//     ties in (row, col) order, compaction.
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <vector>

#include "fsr_common.cuh"

namespace fsr {
namespace ops {

constexpr double kCholQR2Safe = 0.1;   // spectral.CHOLQR2_SAFE
constexpr double kPrecondTol = 0.25;   // spectral.PRECOND_TOL
constexpr double kFusedGramTol = 0.9;  // spectral._precondition_with_gram
constexpr int kHistBits = 12;          // spectral.HIST_BITS

inline double orth_tol(int dt) { return dt == FSR_F64 ? 1e-8 : 1e-4; }  // spectral.ORTH_TOL

// stream-ordered device temporary
struct DevBuf {
  fsr_ctx* ctx = nullptr;
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
  int alloc(fsr_ctx* c, size_t bytes) {
    ctx = c;
    return cuda_status(c, cudaMallocAsync(&p, bytes ? bytes : 1, c->stream), "cudaMallocAsync");
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

std::string& trace_of(fsr_ctx* ctx) {
  static std::mutex mu;
  static std::map<const fsr_ctx*, std::string> traces;
  std::lock_guard<std::mutex> lock(mu);
  return traces[ctx];
}

void trace(fsr_ctx* ctx, const char* fmt, ...) {
  char buf[128];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  std::string& t = trace_of(ctx);
  if (!t.empty()) t += ';';
  t += buf;
}

// one CholeskyQR pass in place: Y <- Y R^-1 (spectral._cholqr_pass)
int cholqr_pass(fsr_ctx* ctx, int dt, int64_t n, int64_t k, void* Y, int64_t ldy, double* G, bool fast_gram,
                bool fast_apply, bool* ok, double* dev) {
  if (fast_gram && dt == FSR_F32)
    FSR_TRY(fsr_gram_levels(ctx, n, k, (const float*)Y, ldy, G, 0, 1));
  else
    FSR_TRY(fsr_gram(ctx, dt, n, k, Y, ldy, G, 0));
  FSR_TRY(fsr_max_offdiag_error(ctx, k, G, dev));
  const int st = fsr_cholesky(ctx, k, G);
  if (st == FSR_ENOTSPD) {
    *ok = false;
    return FSR_OK;
  }
  FSR_TRY(st);
  FSR_TRY(fsr_apply_rinv_levels(ctx, dt, n, k, G, Y, ldy, (fast_gram && fast_apply) ? 1 : 4));
  *ok = true;
  return FSR_OK;
}

int orthonormalize(fsr_ctx* ctx, int dt, int64_t n, int64_t k, void* Y, int64_t ldy, double* G, bool fast_apply) {
  bool ok1 = false, ok2 = false;
  double dev1 = 0.0, dev2 = INFINITY;
  FSR_TRY(cholqr_pass(ctx, dt, n, k, Y, ldy, G, true, fast_apply, &ok1, &dev1));
  if (ok1) FSR_TRY(cholqr_pass(ctx, dt, n, k, Y, ldy, G, false, fast_apply, &ok2, &dev2));
  std::string method = "cholqr2";
  if (!(ok1 && ok2)) {
    FSR_TRY(fsr_householder_qr(ctx, dt, n, k, Y, ldy));
    method = "householder";
    dev2 = INFINITY;
  }
  if (dev2 > kCholQR2Safe) {
    double dev = 0.0;
    FSR_TRY(fsr_gram(ctx, dt, n, k, Y, ldy, G, 0));
    FSR_TRY(fsr_max_offdiag_error(ctx, k, G, &dev));
    if (dev > orth_tol(dt)) {
      FSR_TRY(fsr_householder_qr(ctx, dt, n, k, Y, ldy));
      method += "+householder";
    }
  }
  trace(ctx, "%s", method.c_str());
  return FSR_OK;
}

// Y <- Y R'^-1, span kept, max|Y^T Y - I| <= kPrecondTol (spectral._precondition; fp32)
int precondition(fsr_ctx* ctx, int dt, int64_t n, int64_t k, void* Y, int64_t ldy, double* G, bool fast_apply) {
  bool ok = false;
  double dev = 0.0;
  FSR_TRY(cholqr_pass(ctx, dt, n, k, Y, ldy, G, true, fast_apply, &ok, &dev));
  if (ok) {
    FSR_TRY(fsr_gram_levels(ctx, n, k, (const float*)Y, ldy, G, 0, 1));
    FSR_TRY(fsr_max_offdiag_error(ctx, k, G, &dev));
    if (dev <= kPrecondTol) {
      trace(ctx, "precond(dev=%.3g)", dev);
      return FSR_OK;
    }
    trace(ctx, "precond-failed(dev=%.3g)", dev);
  }
  return orthonormalize(ctx, dt, n, k, Y, ldy, G, fast_apply);
}

// the fused last round: precondition, then the exact Gram G of the result (spectral._precondition_with_gram)
int precondition_with_gram(fsr_ctx* ctx, int dt, int64_t n, int64_t k, void* Y, int64_t ldy, double* G,
                           bool fast_apply) {
  bool ok = false;
  double dev = 0.0;
  FSR_TRY(cholqr_pass(ctx, dt, n, k, Y, ldy, G, true, fast_apply, &ok, &dev));
  if (ok) {
    FSR_TRY(fsr_gram(ctx, dt, n, k, Y, ldy, G, 0));
    FSR_TRY(fsr_max_offdiag_error(ctx, k, G, &dev));
    if (dev <= kFusedGramTol) {
      trace(ctx, "precond+gram(dev=%.3g)", dev);
      return FSR_OK;
    }
    trace(ctx, "precond+gram-failed(dev=%.3g)", dev);
  }
  FSR_TRY(orthonormalize(ctx, dt, n, k, Y, ldy, G, fast_apply));
  return fsr_gram(ctx, dt, n, k, Y, ldy, G, 0);
}

// numpy SeedSequence mixing constants (numpy/random/bit_generator.pyx)
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> 16;
  return v;
}
inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

}  // namespace ops
}  // namespace fsr

using namespace fsr;

extern "C" {

void fsr_philox_key(uint64_t seed, uint64_t* key0, uint64_t* key1) {
  // SeedSequence(seed) with the default pool of 4 words: entropy = seed as
  // little-endian uint32 words, mixed into the pool; generate_state(2, uint64)
  std::vector<uint32_t> ent;
  if (seed == 0) ent.push_back(0);
  for (uint64_t s = seed; s; s >>= 32) ent.push_back((uint32_t)(s & 0xffffffffu));
  uint32_t pool[4];
  uint32_t h = ops::kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = ops::hashmix(i < (int)ent.size() ? ent[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ops::mix(pool[d], ops::hashmix(pool[s], h));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ops::mix(pool[d], ops::hashmix(ent[s], h));
  uint32_t hb = ops::kInitB, w[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= ops::kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  *key0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  *key1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

const char* fsr_schedule_trace(fsr_ctx* ctx) { return ops::trace_of(ctx).c_str(); }

int fsr_orthonormalize(fsr_ctx* ctx, int dtype, int64_t n, int64_t k, void* Y, int64_t ldy) {
  FSR_REQUIRE(ctx, n >= 1 && k >= 1 && k <= n && Y && ldy >= k, "orthonormalize: bad shape");
  ops::trace_of(ctx).clear();
  ops::DevBuf G;
  FSR_TRY(G.alloc(ctx, (size_t)k * k * 8));
  return ops::orthonormalize(ctx, dtype, n, k, Y, ldy, G.as<double>(), true);
}

int fsr_range_finder(fsr_ctx* ctx, int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
                     const void* values, int64_t r_hat, int q, uint64_t seed, int flags, void* Q, void* B,
                     double* gram_out, int* gram_valid) {
  FSR_REQUIRE(ctx, r_hat >= 1 && r_hat <= n, "r_hat must lie in [1, n], got %lld for n=%lld", (long long)r_hat,
              (long long)n);
  FSR_REQUIRE(ctx, q >= 1, "q must be at least 1");
  FSR_REQUIRE(ctx, indptr && Q && B && (dtype == FSR_F32 || dtype == FSR_F64), "range_finder: bad arguments");
  ops::trace_of(ctx).clear();
  const bool span_only = (flags & FSR_SI_SPAN_ONLY) && dtype == FSR_F32;
  const bool fused = span_only && (flags & FSR_SI_FUSED_RR) && gram_out;
  const bool fast_apply = flags & FSR_SI_FAST_FIRST_APPLY;
  if (gram_valid) *gram_valid = fused ? 1 : 0;
  ops::DevBuf Gs;
  FSR_TRY(Gs.alloc(ctx, (size_t)r_hat * r_hat * 8));
  double* G = Gs.as<double>();
  // the rounds alternate between the two caller blocks; start where the last
  // processed basis lands in Q and the last product in B
  void* X[2] = {(q % 2) ? Q : B, (q % 2) ? B : Q};
  uint64_t k0, k1;
  fsr_philox_key(seed, &k0, &k1);
  FSR_TRY(fsr_gaussian_block(ctx, dtype, n, r_hat, 0, n, k0, k1, X[0]));
  for (int t = 0; t < q; ++t) {
    void* Y = X[t & 1];
    if (t == q - 1 && fused) {
      FSR_TRY(ops::precondition_with_gram(ctx, dtype, n, r_hat, Y, r_hat, G, fast_apply));
      FSR_CUDA(ctx, cudaMemcpyAsync(gram_out, G, (size_t)r_hat * r_hat * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    } else if (span_only && t < q - 1) {
      if (t > 0 || 4 * r_hat > n)
        FSR_TRY(ops::precondition(ctx, dtype, n, r_hat, Y, r_hat, G, fast_apply));
      else
        ops::trace(ctx, "start");
    } else {
      FSR_TRY(ops::orthonormalize(ctx, dtype, n, r_hat, Y, r_hat, G, fast_apply));
    }
    FSR_TRY(fsr_csr_spmm(ctx, dtype, n, indptr, indices, values, r_hat, Y, r_hat, X[(t + 1) & 1], r_hat));
  }
  return FSR_OK;
}

int fsr_rayleigh_ritz(fsr_ctx* ctx, int dtype, int64_t n, int64_t r_hat, const void* Q, int64_t ldq, const void* B,
                      int64_t ldb, const double* gram, int64_t r, double* lam_host, void* U, int64_t ldu,
                      double* eta) {
  FSR_REQUIRE(ctx, r >= 1 && r <= r_hat, "r must lie in [1, r_hat=%lld], got %lld", (long long)r_hat, (long long)r);
  FSR_REQUIRE(ctx, n >= 1 && Q && B && lam_host && U && eta && ldq >= r_hat && ldb >= r_hat && ldu >= r,
              "rayleigh_ritz: bad arguments");
  ops::DevBuf C, V, G2, best;
  FSR_TRY(C.alloc(ctx, (size_t)r_hat * r_hat * 8));
  FSR_TRY(V.alloc(ctx, (size_t)r_hat * r * 8));
  FSR_TRY(fsr_cross_sym(ctx, dtype, n, r_hat, Q, ldq, B, ldb, C.as<double>(), 0));
  if (gram) {  // sygvd destroys G: work on a copy
    FSR_TRY(G2.alloc(ctx, (size_t)r_hat * r_hat * 8));
    FSR_CUDA(ctx, cudaMemcpyAsync(G2.p, gram, (size_t)r_hat * r_hat * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    FSR_TRY(fsr_eigh_gen_desc(ctx, r_hat, C.as<double>(), G2.as<double>(), r, lam_host, V.as<double>()));
  } else {
    FSR_TRY(fsr_eigh_desc(ctx, r_hat, C.as<double>(), r, lam_host, V.as<double>()));
  }
  FSR_TRY(fsr_lift(ctx, dtype, n, r_hat, r, Q, ldq, V.as<double>(), U, ldu));
  FSR_TRY(best.alloc(ctx, (size_t)r * 24));
  double* best_abs = best.as<double>();
  int64_t* best_row = (int64_t*)(best_abs + r);
  double* best_val = (double*)(best_row + r);
  FSR_TRY(fsr_col_absmax(ctx, dtype, n, r, U, ldu, 0, best_abs, best_row, best_val));
  return fsr_apply_signs_rownorm(ctx, dtype, n, r, U, ldu, best_val, eta);
}

int fsr_decompose(fsr_ctx* ctx, int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
                  const void* values, int64_t r, int64_t p, int q, uint64_t seed, int flags, double* lam_host,
                  void* U, int64_t ldu, double* eta) {
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && p >= 0, "decompose: need n >= 1, r >= 1, p >= 0");
  const int64_t r_hat = std::min<int64_t>(r + p, n);
  FSR_REQUIRE(ctx, r <= r_hat, "r=%lld exceeds n=%lld", (long long)r, (long long)n);
  const size_t es = dtype_size(dtype);
  ops::DevBuf Q, B, G;
  FSR_TRY(Q.alloc(ctx, (size_t)n * r_hat * es));
  FSR_TRY(B.alloc(ctx, (size_t)n * r_hat * es));
  FSR_TRY(G.alloc(ctx, (size_t)r_hat * r_hat * 8));
  int gram_valid = 0;
  FSR_TRY(fsr_range_finder(ctx, dtype, n, indptr, indices, values, r_hat, q, seed, flags, Q.p, B.p, G.as<double>(),
                           &gram_valid));
  return fsr_rayleigh_ritz(ctx, dtype, n, r_hat, Q.p, r_hat, B.p, r_hat, gram_valid ? G.as<double>() : nullptr, r,
                           lam_host, U, ldu, eta);
}

int fsr_sparsify_select(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, int64_t tau,
                        uint64_t* T_out, int64_t* ties_out, int64_t* keep_out) {
  FSR_REQUIRE(ctx, tau >= 1, "tau must be positive");
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && U && ldu >= r && T_out && ties_out && keep_out, "sparsify_select: bad arguments");
  const int kb = dtype == FSR_F64 ? 63 : 31;
  ops::DevBuf hd;
  FSR_TRY(hd.alloc(ctx, (size_t)8 << ops::kHistBits));
  std::vector<uint64_t> h((size_t)1 << ops::kHistBits);
  auto hist = [&](uint64_t prefix, int shift, int bits) -> int {
    FSR_CUDA(ctx, cudaMemsetAsync(hd.p, 0, (size_t)8 << bits, ctx->stream));
    FSR_TRY(fsr_abs_histogram(ctx, dtype, n, r, U, ldu, prefix, shift, bits, hd.as<uint64_t>()));
    FSR_CUDA(ctx, cudaMemcpyAsync(h.data(), hd.p, (size_t)8 << bits, cudaMemcpyDeviceToHost, ctx->stream));
    FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return FSR_OK;
  };
  int shift = kb - ops::kHistBits, bits = ops::kHistBits;
  FSR_TRY(hist(0, shift, bits));
  int64_t nnz = 0;
  for (int i = 0; i < (1 << bits); ++i) nnz += (int64_t)h[i];
  const int64_t keep = std::min<int64_t>(tau, nnz);
  *keep_out = keep;
  if (keep == nnz) {
    *T_out = 0;
    *ties_out = 0;
    return FSR_OK;
  }
  int64_t need = keep;
  uint64_t prefix = 0;
  for (;;) {  // spectral.select_threshold: the digit whose top-down cumulative count reaches `need`
    int64_t cum = 0;
    int b = (1 << bits) - 1;
    for (; b >= 0; --b) {
      if (cum + (int64_t)h[b] >= need) break;
      cum += (int64_t)h[b];
    }
    need -= cum;
    prefix |= (uint64_t)b << shift;
    if (shift == 0) {
      *T_out = prefix;
      *ties_out = need;
      return FSR_OK;
    }
    bits = std::min(ops::kHistBits, shift);
    shift -= bits;
    FSR_TRY(hist(prefix, shift, bits));
  }
}

int fsr_sparsify(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, int64_t tau,
                 int64_t* indptr_out, int32_t* indices_out, void* values_out, int64_t capacity, double* eta,
                 int64_t* nnz_host) {
  FSR_REQUIRE(ctx, indptr_out && indices_out && values_out && eta && nnz_host, "sparsify: missing outputs");
  uint64_t T = 0;
  int64_t ties = 0, keep = 0;
  FSR_TRY(fsr_sparsify_select(ctx, dtype, n, r, U, ldu, tau, &T, &ties, &keep));
  FSR_REQUIRE(ctx, capacity >= keep, "sparsify: capacity %lld below the kept count %lld", (long long)capacity,
              (long long)keep);
  return fsr_sparsify_apply(ctx, dtype, n, r, U, ldu, T, ties, indptr_out, indices_out, values_out, eta, nnz_host);
}

int fsr_sparsify_apply(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, const void* U, int64_t ldu, uint64_t T,
                       int64_t ties, int64_t* indptr_out, int32_t* indices_out, void* values_out, double* eta,
                       int64_t* nnz_host) {
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && U && ldu >= r && ties >= 0, "sparsify_apply: bad arguments");
  FSR_REQUIRE(ctx, indptr_out && indices_out && values_out && eta && nnz_host, "sparsify_apply: missing outputs");
  ops::DevBuf cnt;
  FSR_TRY(cnt.alloc(ctx, (size_t)n * 16));
  int64_t* gt = cnt.as<int64_t>();
  int64_t* eq = gt + n;
  FSR_TRY(fsr_threshold_counts(ctx, dtype, n, r, U, ldu, T, gt, eq));
  return fsr_threshold_compact(ctx, dtype, n, r, U, ldu, T, 0, ties, gt, eq, indptr_out, indices_out, values_out, eta,
                               nnz_host);
}

}  // extern "C"
