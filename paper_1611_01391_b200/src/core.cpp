// Host containers, Rng, status mapping and the device context.
// Rng restates /root/reference/proj/src/rng.cpp:8-66 bit for bit.
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>
#include <numbers>
#include <string>

#include "slra/devbuf.hpp"
#include "slra/errors.hpp"
#include "slra/matrix.hpp"
#include "slra/rng.hpp"

namespace slra {

// ---------------------------------------------------------------- status
void check(int status, const char* where) {
  if (status == SLRA_OK) return;
  const std::string msg = std::string(where) + ": " + slra_status_string(status);
  switch (status) {
    case SLRA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SLRA_ERR_RANGE_FAILURE: throw RangeFailure(msg);
    case SLRA_ERR_SKETCH_RANK_FAILURE: throw SketchRankFailure(msg);
    case SLRA_ERR_SELECTION_FAILURE: throw SelectionFailure(msg);
    case SLRA_ERR_GENERATOR_RANK_FAILURE: throw GeneratorRankFailure(msg);
    case SLRA_ERR_PREMULT_RANK_FAILURE: throw PremultRankFailure(msg);
    case SLRA_ERR_UNSUPPORTED: throw std::invalid_argument(msg);
    default: throw DeviceError(msg + " (" + slra_last_error() + ")");
  }
}

// ---------------------------------------------------------------- context
namespace {
std::mutex g_mu;
slra_ctx g_ctx = nullptr;
std::vector<void (*)()>* g_hooks = new std::vector<void (*)()>();
}  // namespace

slra_ctx device_context() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx) check(slra_ctx_create(0, nullptr, &g_ctx), "slra_ctx_create");
  return g_ctx;
}

void on_context_release(void (*hook)()) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_hooks->push_back(hook);
}

void set_device(int device, void* stream) {
  std::vector<void (*)()> hooks;
  bool live = false;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    hooks = *g_hooks;
    live = g_ctx != nullptr;
  }
  if (live)
    for (auto f : hooks) f();
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx) slra_ctx_destroy(g_ctx);
  g_ctx = nullptr;
  check(slra_ctx_create(device, stream, &g_ctx), "slra_ctx_create");
}

// ---------------------------------------------------------------- Matrix
Matrix Matrix::Identity(Index rows, Index cols) {
  Matrix I(rows, cols);
  for (Index i = 0; i < std::min(rows, cols); ++i) I(i, i) = 1.0;
  return I;
}

Matrix Matrix::transpose() const {
  Matrix T(c_, r_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) T(j, i) = (*this)(i, j);
  return T;
}

IndexSet::IndexSet(std::vector<Index> idx, Index bound) : idx_(std::move(idx)), bound_(bound) {
  std::vector<bool> seen(static_cast<size_t>(bound), false);
  for (Index i : idx_) {
    if (i < 0 || i >= bound) throw std::invalid_argument("IndexSet: index out of bound");
    if (seen[static_cast<size_t>(i)]) throw std::invalid_argument("IndexSet: duplicate index");
    seen[static_cast<size_t>(i)] = true;
  }
}

IndexSet IndexSet::iota(Index count, Index bound) {
  std::vector<Index> v(static_cast<size_t>(count));
  for (Index i = 0; i < count; ++i) v[static_cast<size_t>(i)] = i;
  return IndexSet(std::move(v), bound);
}

bool IndexSet::contains(Index i) const {
  for (Index j : idx_)
    if (j == i) return true;
  return false;
}

// ---------------------------------------------------------------- DeviceMatrix
DeviceMatrix::DeviceMatrix(Index rows, Index cols) : r_(rows), c_(cols), ld_(rows > 0 ? rows : 1), owns_(true) {
  void* p = nullptr;
  check(slra_device_alloc(device_context(), 8 * std::max<Index>(1, rows * cols), &p), "DeviceMatrix");
  p_ = static_cast<double*>(p);
}

DeviceMatrix DeviceMatrix::upload(const Matrix& M) {
  DeviceMatrix d(M.rows(), M.cols());
  check(slra_memcpy_h2d(device_context(), d.p_, M.data(), 8 * M.size()), "DeviceMatrix::upload");
  return d;
}

DeviceMatrix DeviceMatrix::view(double* ptr, Index rows, Index cols, Index ld) {
  DeviceMatrix d;
  d.r_ = rows;
  d.c_ = cols;
  d.ld_ = ld;
  d.p_ = ptr;
  d.owns_ = false;
  return d;
}

DeviceMatrix& DeviceMatrix::operator=(DeviceMatrix&& o) noexcept {
  if (this != &o) {
    if (owns_ && p_) slra_device_free(device_context(), p_);
    r_ = o.r_;
    c_ = o.c_;
    ld_ = o.ld_;
    p_ = o.p_;
    owns_ = o.owns_;
    o.p_ = nullptr;
    o.owns_ = false;
  }
  return *this;
}

DeviceMatrix::~DeviceMatrix() {
  if (owns_ && p_) slra_device_free(device_context(), p_);  // stream-ordered: no sync
}

Matrix DeviceMatrix::download() const {
  Matrix M(r_, c_);
  if (r_ == 0 || c_ == 0) return M;
  if (ld_ == r_) {
    check(slra_memcpy_d2h(device_context(), M.data(), p_, 8 * r_ * c_), "DeviceMatrix::download");
  } else {
    for (Index j = 0; j < c_; ++j)
      check(slra_memcpy_d2h(device_context(), M.data() + j * r_, p_ + j * ld_, 8 * r_), "DeviceMatrix::download");
  }
  return M;
}

// select_* are host-side copies of host matrices (linalg.cpp:35-52); the
// device path gathers with slra_gather_* instead.
Matrix select_rows(const Matrix& A, const IndexSet& I) {
  Matrix out(I.size(), A.cols());
  for (Index j = 0; j < A.cols(); ++j)
    for (Index t = 0; t < I.size(); ++t) out(t, j) = A(I[t], j);
  return out;
}
Matrix select_cols(const Matrix& A, const IndexSet& J) {
  Matrix out(A.rows(), J.size());
  for (Index t = 0; t < J.size(); ++t)
    for (Index i = 0; i < A.rows(); ++i) out(i, t) = A(i, J[t]);
  return out;
}
Matrix select_block(const Matrix& A, const IndexSet& I, const IndexSet& J) {
  Matrix out(I.size(), J.size());
  for (Index s = 0; s < I.size(); ++s)
    for (Index t = 0; t < J.size(); ++t) out(s, t) = A(I[s], J[t]);
  return out;
}

// ---------------------------------------------------------------- Rng (rng.cpp:8-66)
double Rng::gaussian() {
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}

Index Rng::uniform_index(Index n) {
  const std::uint64_t un = static_cast<std::uint64_t>(n);
  const std::uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  std::uint64_t x = next_u64();
  while (x >= limit) x = next_u64();
  return static_cast<Index>(x % un);
}

std::vector<Index> Rng::permutation(Index n) {
  std::vector<Index> p(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) p[static_cast<size_t>(i)] = i;
  for (Index i = n - 1; i > 0; --i) std::swap(p[static_cast<size_t>(i)], p[static_cast<size_t>(uniform_index(i + 1))]);
  return p;
}

std::vector<Index> Rng::distinct_indices(Index k, Index n) {
  std::vector<Index> pool(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) pool[static_cast<size_t>(i)] = i;
  std::vector<Index> out;
  out.reserve(static_cast<size_t>(k));
  for (Index t = 0; t < k; ++t) {
    const Index j = t + uniform_index(n - t);
    std::swap(pool[static_cast<size_t>(t)], pool[static_cast<size_t>(j)]);
    out.push_back(pool[static_cast<size_t>(t)]);
  }
  return out;
}

Matrix Rng::gaussian_matrix(Index rows, Index cols) {
  Matrix G(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) G(i, j) = gaussian();
  return G;
}

Vector Rng::gaussian_vector(Index n) {
  Vector v(static_cast<size_t>(n));
  for (auto& x : v) x = gaussian();
  return v;
}

std::uint64_t Rng::derive_seed(std::uint64_t master, std::uint64_t stream) {
  std::uint64_t z = master + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace slra
