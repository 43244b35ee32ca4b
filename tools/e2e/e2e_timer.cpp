// BENCH INFRASTRUCTURE (not product code): host-clock timing of the
// host-buffer C-ABI entry desmoe_layer_forward_host (include/desmoe.h), the
// call a C/C++ user of the drop-in makes. Each call is bracketed by
// std::chrono::steady_clock reads in C, so neither the Python/ctypes
// trampoline nor a CUDA event recorded after the call returns (which would add
// the stream's submission latency to a result the host already holds) is
// inside the measurement. The call itself copies the caller's pinned x in,
// runs the layer and returns once y (fp32) and the stats are visible in host
// memory.
#include <chrono>

#include "desmoe.h"

extern "C" int e2e_time_host_calls(desmoe_ctx* const* ctxs, desmoe_experts* const* experts,
                                   const void* const* w_routers, int layers,
                                   const void* const* xs, int nx, int n,
                                   const desmoe_route_cfg* cfg, float* y_host, int* stats_host,
                                   void* stream, int calls, double* us_out) {
  for (int i = 0; i < calls; ++i) {
    const int l = i % layers;
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = desmoe_layer_forward_host(ctxs[l], experts[l], w_routers[l], xs[i % nx], n, cfg,
                                             y_host, stats_host, stream);
    const auto t1 = std::chrono::steady_clock::now();
    if (rc) return rc;
    us_out[i] = std::chrono::duration<double, std::micro>(t1 - t0).count();
  }
  return 0;
}
