#pragma once
// Per-thread CUDA context of the C++ facade: every ranger:: compute function
// runs on the GPU through include/ranger_cuda.h.  The device is RG_DEVICE
// (default 0).  There is no CPU fallback: a missing GPU or library throws.
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../ranger_cuda.h"

namespace ranger::cuda {

class Context {
 public:
  Context() {
    const char* env = std::getenv("RG_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    if (rg_ctx_create(dev, &ctx_) != RG_OK)
      throw std::runtime_error(std::string("ranger: CUDA context unavailable: ") + rg_create_error());
  }
  ~Context() { rg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rg_ctx* get() const { return ctx_; }

 private:
  rg_ctx* ctx_ = nullptr;
};

inline rg_ctx* ctx() {
  thread_local Context c;
  return c.get();
}

// Map a status to the reference's exception types.
inline void check(rg_status st) {
  if (st == RG_OK) return;
  const std::string msg = rg_last_error(ctx());
  if (st == RG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("ranger CUDA error: " + msg);
}

}  // namespace ranger::cuda
