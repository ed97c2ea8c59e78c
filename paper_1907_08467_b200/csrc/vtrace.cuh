// vtrace.cuh — batched V-trace targets (Eqs.
// target.off / rho / c and the recursive form "we compute the V-trace update recursively").
//
// One thread per trajectory (env) b, walking t = T-1 .. 0 with the recursive form
//   v_t = V_t + delta_t + gamma_t c_t (v_{t+1} - V_{t+1}),   v_T = V_boot,
//   delta_t = rho_t (r_t + gamma_t V_{t+1} - V_t),  rho_t = min(rho_bar, pi/mu), c_t = min(c_bar, pi/mu),
// with gamma_t = gamma (1 - done_t) (a terminal at step t stops bootstrapping through it,
// DESIGN.md R#33), and the policy-gradient advantage r_t + gamma_t v_{t+1} - V_t.  Arrays are
// time-major [T][B], so a warp's 32 trajectories read and write 128 contiguous bytes per array
// and step: the kernel is a pure HBM stream, fp32 in and out, fp32 arithmetic.
#pragma once
#include <stdint.h>

namespace cule {

__global__ void __launch_bounds__(64) vtrace_kernel(const float* __restrict__ r, const float* __restrict__ V,
                                                     const float* __restrict__ V_boot,
                                                     const float* __restrict__ log_mu,
                                                     const float* __restrict__ log_pi,
                                                     const uint8_t* __restrict__ done, uint32_t T, uint32_t B,
                                                     float gamma, float rho_bar, float c_bar, float* __restrict__ vs,
                                                     float* __restrict__ rho_out, float* __restrict__ adv) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float v_next = V_boot[b];  // v_{t+1}
  float V_next = v_next;     // V(s_{t+1})
  // the recursion is sequential in t but its inputs are not: each chunk of kChunk steps is
  // loaded first (all loads in flight together), then walked backwards
  constexpr uint32_t kChunk = 8;
  for (uint32_t hi = T; hi > 0;) {
    const uint32_t lo = hi > kChunk ? hi - kChunk : 0u;
    float rr[kChunk], vv[kChunk], lm[kChunk], lp[kChunk];
    uint8_t dd[kChunk];
#pragma unroll
    for (uint32_t j = 0; j < kChunk; ++j) {
      if (lo + j < hi) {
        const size_t o = (size_t)(lo + j) * B + b;
        rr[j] = r[o]; vv[j] = V[o]; lm[j] = log_mu[o]; lp[j] = log_pi[o]; dd[j] = done[o];
      }
    }
#pragma unroll
    for (int j = kChunk - 1; j >= 0; --j) {
      if (lo + (uint32_t)j >= hi) continue;
      const size_t o = (size_t)(lo + (uint32_t)j) * B + b;
      const float ratio = expf(lp[j] - lm[j]);
      const float rho = fminf(rho_bar, ratio), c = fminf(c_bar, ratio);
      const float g = dd[j] ? 0.0f : gamma;
      const float Vt = vv[j], rt = rr[j];
      const float delta = rho * (rt + g * V_next - Vt);
      const float v = Vt + delta + g * c * (v_next - V_next);
      vs[o] = v;
      rho_out[o] = rho;
      adv[o] = rt + g * v_next - Vt;
      v_next = v;
      V_next = Vt;
    }
    hi = lo;
  }
}

}  // namespace cule
