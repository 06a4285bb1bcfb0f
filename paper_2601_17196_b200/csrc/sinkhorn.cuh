// sinkhorn.cuh — extended (dummy-node) log-domain Sinkhorn (solvers.hpp:387-589).
// Included by capi.cu after the Session base.
#pragma once

namespace potgpu {

inline std::unique_ptr<Session> make_sinkhorn_session(Context&, int, int64_t) {
  throw Error(POTGPU_ERR_UNSUPPORTED, "sinkhorn solvers: not built yet");
}

}  // namespace potgpu
