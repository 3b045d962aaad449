// placeholder until the tcgen05 backward lands
#include <cuda_runtime.h>
#include "ttt_params.cuh"
namespace tttk {
cudaError_t launch_bwd_sm100(const Params&, const BwdMaps&, cudaStream_t) { return cudaErrorNotSupported; }
}
