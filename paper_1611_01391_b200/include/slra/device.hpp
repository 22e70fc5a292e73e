// Process-wide device context used by the host entry points. One context per
// (device, stream); the default is device 0 on a context-owned stream.
#pragma once

#include <cstdint>

#include "slra_cuda.h"

namespace slra {

/// The context every host entry point runs on. Creating it fails loudly
/// (DeviceError) when no sm_100 device is usable — there is no CPU path.
slra_ctx device_context();
/// Re-target the default context (e.g. torch's current device/stream).
/// Registered release hooks run first, while the old context is still
/// current, so buffers tied to it are freed through it.
void set_device(int device, void* stream = nullptr);
void on_context_release(void (*hook)());

}  // namespace slra
