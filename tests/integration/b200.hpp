// the reference-side glue — one shared context and the
// status -> typed-exception mapping (slra_cuda.h status codes 1:1 onto
// errors.hpp:11-33) — as a maintainer would add it (proj/src/b200.hpp).
#pragma once
#include <stdexcept>
#include <string>

#include "slra_cuda.h"

namespace slra::b200 {
inline slra_ctx ctx() {  // one context per process
  static slra_ctx c = [] {
    slra_ctx x{};
    if (slra_ctx_create(0, nullptr, &x) != SLRA_OK) throw std::runtime_error("slra_b200: no sm_100 device");
    return x;
  }();
  return c;
}
inline void check(int st, const char* what) {
  switch (st) {
    case SLRA_OK: return;
    case SLRA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(what);
    case SLRA_ERR_RANGE_FAILURE: throw RangeFailure(what);
    case SLRA_ERR_SKETCH_RANK_FAILURE: throw SketchRankFailure(what);
    case SLRA_ERR_SELECTION_FAILURE: throw SelectionFailure(what);
    case SLRA_ERR_GENERATOR_RANK_FAILURE: throw GeneratorRankFailure(what);
    case SLRA_ERR_PREMULT_RANK_FAILURE: throw PremultRankFailure(what);
    default: throw std::runtime_error(std::string(what) + ": " + slra_status_string(st));
  }
}
struct Dev {  // RAII device buffer
  void* p = nullptr;
  explicit Dev(size_t bytes) { check(slra_device_alloc(ctx(), (int64_t)bytes, &p), "alloc"); }
  ~Dev() { slra_device_free(ctx(), p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
}  // namespace slra::b200
