// K9 Adam (sm_100a): replaces AdamState::step (adam.hpp:55-101) and the
// densification statistics update (gradient.hpp:39-45, trainer.hpp:189-193):
// one pass over the planar fp32 params/grads/moments, quaternion
// renormalisation and log-scale clamp fused in (adam_math.cuh). dsg_train
// runs the same update inside the chain kernel instead (chain.cu); this
// launch serves dsg_adam_step and steps with nothing visible.
#include "dsg_internal.h"
#include "raster.h"
#include "adam_math.cuh"

namespace dsg {

namespace {

#ifndef DSG_ADAM_MINB
#define DSG_ADAM_MINB 1
#endif
__global__ void __launch_bounds__(256, DSG_ADAM_MINB) k_adam(AdamArgs a) {
  DSG_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const float* __restrict__ G = a.grads;
  const int64_t P = a.pitch;
  adam_splat(a, i, [&](int k) { return __ldg(G + k * P + i); }, a.touch[i] > 0, a.dmean[i],
             a.dmean[P + i]);
}

}  // namespace

void adam_update(const AdamArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  pdl_launch(k_adam, (unsigned)((a.n + 255) / 256), 256, 0, st, a);
  count_launch();
  DSG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace dsg
