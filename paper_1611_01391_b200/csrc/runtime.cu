// Context, memory and status plumbing for slra_cuda.h. No CPU fallback:
// without a usable sm_100 device every entry point fails with
// SLRA_ERR_NO_DEVICE.
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace slra_dev {

static thread_local std::string g_last_error;

void set_last_error(const std::string& s) { g_last_error = s; }

int cuda_status(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorNoKernelImageForDevice)
    return SLRA_ERR_NO_DEVICE;
  return SLRA_ERR_CUDA;
}

void* workspace(Context* c, size_t bytes) {
  if (bytes <= c->ws_bytes) return c->ws;
  cudaStreamSynchronize(c->stream);
  if (c->ws) cudaFree(c->ws);
  size_t want = bytes + bytes / 4 + (1 << 20);
  if (cudaMalloc(&c->ws, want) != cudaSuccess) {
    c->ws = nullptr;
    c->ws_bytes = 0;
    return nullptr;
  }
  c->ws_bytes = want;
  return c->ws;
}

void* pinned_scratch(Context* c, size_t bytes) {
  if (bytes <= c->pinned_bytes) return c->pinned;
  cudaStreamSynchronize(c->stream);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (cudaMallocHost(&c->pinned, bytes + 4096) != cudaSuccess) {
    c->pinned = nullptr;
    c->pinned_bytes = 0;
    return nullptr;
  }
  c->pinned_bytes = bytes + 4096;
  return c->pinned;
}

double* partials(Context* c, int n) {
  if (n <= c->partials_cap) return c->partials;
  cudaStreamSynchronize(c->stream);
  if (c->partials) cudaFree(c->partials);
  if (cudaMalloc(&c->partials, sizeof(double) * (n + 64)) != cudaSuccess) {
    c->partials = nullptr;
    c->partials_cap = 0;
    return nullptr;
  }
  c->partials_cap = n + 64;
  return c->partials;
}

void* arena(Context* c, int slot, size_t bytes) {
  if (bytes <= c->arena_bytes[slot]) return c->arena[slot];
  cudaStreamSynchronize(c->stream);
  if (c->arena[slot]) cudaFree(c->arena[slot]);
  const size_t want = bytes + bytes / 8 + 4096;
  if (cudaMalloc(&c->arena[slot], want) != cudaSuccess) {
    c->arena[slot] = nullptr;
    c->arena_bytes[slot] = 0;
    return nullptr;
  }
  c->arena_bytes[slot] = want;
  return c->arena[slot];
}

cudaEvent_t pooled_event(Context* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

const char* slra_status_string(int s) {
  switch (s) {
    case SLRA_OK: return "ok";
    case SLRA_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SLRA_ERR_RANGE_FAILURE: return "range_finder: sketch M H has numerical rank below target";
    case SLRA_ERR_SKETCH_RANK_FAILURE: return "sketch_solve: sketched matrix FA is rank deficient";
    case SLRA_ERR_SELECTION_FAILURE: return "maxvol_rows: singular pivot block";
    case SLRA_ERR_GENERATOR_RANK_FAILURE: return "primitive_cur: generator rank below target";
    case SLRA_ERR_PREMULT_RANK_FAILURE: return "lra_premult: F U has numerical rank below target";
    case SLRA_ERR_CUDA: return "CUDA error";
    case SLRA_ERR_NO_DEVICE: return "no usable CUDA device (sm_100a required)";
    case SLRA_ERR_UNSUPPORTED: return "shape not supported by the device kernels";
    default: return "unknown status";
  }
}

const char* slra_last_error(void) { return g_last_error.c_str(); }

int slra_ctx_create(int device, void* stream, slra_ctx* out) {
  if (!out) return SLRA_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_last_error(e != cudaSuccess ? cudaGetErrorString(e) : "no CUDA device");
    return SLRA_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= n) return SLRA_ERR_INVALID_ARGUMENT;
  cudaDeviceProp prop;
  SLRA_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_last_error("device is not sm_100 (Blackwell B200)");
    return SLRA_ERR_NO_DEVICE;
  }
  SLRA_CUDA(cudaSetDevice(device));
  auto* c = new Context();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return SLRA_ERR_CUDA;
    }
    c->owns_stream = true;
  }
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // keep freed blocks for reuse
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (cudaMalloc(&c->dsmall, 4096) != cudaSuccess || cudaMallocHost(&c->hsmall, 4096) != cudaSuccess) {
    delete c;
    return SLRA_ERR_CUDA;
  }
  *out = reinterpret_cast<slra_ctx>(c);
  return SLRA_OK;
}

int slra_ctx_destroy(slra_ctx ctx) {
  Context* c = C(ctx);
  if (!c) return SLRA_OK;
  cudaStreamSynchronize(c->stream);
  if (c->ws) cudaFree(c->ws);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->partials) cudaFree(c->partials);
  if (c->dsmall) cudaFree(c->dsmall);
  for (int i = 0; i < kArenaSlots; ++i)
    if (c->arena[i]) cudaFree(c->arena[i]);
  for (auto& r : c->records) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->hsmall) cudaFreeHost(c->hsmall);
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->owns_stream) cudaStreamDestroy(c->stream);
  delete c;
  return SLRA_OK;
}

int slra_ctx_synchronize(slra_ctx ctx) {
  SLRA_CUDA(cudaStreamSynchronize(C(ctx)->stream));
  return SLRA_OK;
}

void* slra_ctx_stream(slra_ctx ctx) { return C(ctx)->stream; }

int64_t slra_ctx_launch_count(slra_ctx ctx) { return C(ctx)->launches; }

int slra_ctx_set_timing(slra_ctx ctx, int on) {
  Context* c = C(ctx);
  SLRA_CUDA(cudaStreamSynchronize(c->stream));
  for (auto& r : c->records) {
    c->event_pool.push_back(r.start);
    c->event_pool.push_back(r.stop);
  }
  c->records.clear();
  c->timing = on != 0;
  return SLRA_OK;
}

int slra_ctx_timing_report(slra_ctx ctx, char* buf, int64_t len) {
  Context* c = C(ctx);
  SLRA_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<std::string> fams;
  std::vector<double> ms;
  std::vector<int64_t> cnt;
  for (auto& r : c->records) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.start, r.stop);
    size_t i = 0;
    while (i < fams.size() && fams[i] != r.family) ++i;
    if (i == fams.size()) {
      fams.push_back(r.family);
      ms.push_back(0.0);
      cnt.push_back(0);
    }
    ms[i] += t;
    cnt[i] += 1;
  }
  std::string out;
  for (size_t i = 0; i < fams.size(); ++i) {
    char tmp[160];
    snprintf(tmp, sizeof(tmp), "%s%s=%.6f,%lld", i ? ";" : "", fams[i].c_str(), ms[i], (long long)cnt[i]);
    out += tmp;
  }
  if (buf && len > 0) {
    strncpy(buf, out.c_str(), (size_t)len - 1);
    buf[len - 1] = 0;
  }
  return SLRA_OK;
}

// Stream-ordered allocations from the device's default pool (release
// threshold raised at context creation): the host layer's many short-lived
// operands cost no cudaMalloc/cudaFree round trip and no device sync.
int slra_device_alloc(slra_ctx ctx, int64_t bytes, void** d_out) {
  if (!ctx || !d_out || bytes < 0) return SLRA_ERR_INVALID_ARGUMENT;
  SLRA_CUDA(cudaMallocAsync(d_out, bytes > 0 ? bytes : 8, C(ctx)->stream));
  return SLRA_OK;
}

int slra_device_free(slra_ctx ctx, void* p) {
  if (!ctx) return SLRA_ERR_INVALID_ARGUMENT;
  if (p) SLRA_CUDA(cudaFreeAsync(p, C(ctx)->stream));
  return SLRA_OK;
}

int slra_memcpy_h2d(slra_ctx ctx, void* d, const void* h, int64_t bytes) {
  if (bytes <= 0) return SLRA_OK;
  SLRA_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, C(ctx)->stream));
  return SLRA_OK;
}

int slra_memcpy_d2h(slra_ctx ctx, void* h, const void* d, int64_t bytes) {
  if (bytes <= 0) return SLRA_OK;
  SLRA_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, C(ctx)->stream));
  SLRA_CUDA(cudaStreamSynchronize(C(ctx)->stream));
  return SLRA_OK;
}

int slra_host_alloc(int64_t bytes, void** h_out) {
  if (!h_out || bytes < 0) return SLRA_ERR_INVALID_ARGUMENT;
  *h_out = nullptr;
  if (bytes == 0) return SLRA_OK;
  SLRA_CUDA(cudaHostAlloc(h_out, (size_t)bytes, cudaHostAllocDefault));
  return SLRA_OK;
}

int slra_host_free(void* h) {
  if (h) SLRA_CUDA(cudaFreeHost(h));
  return SLRA_OK;
}

int slra_memcpy_d2d(slra_ctx ctx, void* d, const void* s, int64_t bytes) {
  if (bytes <= 0) return SLRA_OK;
  SLRA_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, C(ctx)->stream));
  return SLRA_OK;
}

}  // extern "C"
