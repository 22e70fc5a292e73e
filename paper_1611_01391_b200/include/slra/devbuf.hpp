// RAII device buffer over the C-ABI allocator (host code never includes CUDA).
#pragma once

#include <vector>

#include "slra/device.hpp"
#include "slra/errors.hpp"

namespace slra {

template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) : n_(n) {
    void* p = nullptr;
    check(slra_device_alloc(device_context(), static_cast<int64_t>(sizeof(T) * (n ? n : 1)), &p), "DevBuf");
    p_ = static_cast<T*>(p);
  }
  explicit DevBuf(const std::vector<T>& h) : DevBuf(h.size()) { upload(h); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (p_) slra_device_free(device_context(), p_);
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
    }
    return *this;
  }
  ~DevBuf() {
    if (p_) slra_device_free(device_context(), p_);  // stream-ordered: no sync
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const std::vector<T>& h) {
    check(slra_memcpy_h2d(device_context(), p_, h.data(), static_cast<int64_t>(sizeof(T) * h.size())), "DevBuf::upload");
  }
  std::vector<T> download() const {
    std::vector<T> h(n_);
    check(slra_memcpy_d2h(device_context(), h.data(), p_, static_cast<int64_t>(sizeof(T) * n_)), "DevBuf::download");
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace slra
