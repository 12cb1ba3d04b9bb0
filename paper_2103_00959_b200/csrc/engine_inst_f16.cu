// engine_inst_f16.cu -- explicit instantiations of the row-gather engine with
// fp16 feature storage (XF16, spmm_engine.cuh) for gsp_spmm_f16.
#define GSP_ENGINE_INSTANTIATE
#include "spmm_engine.cuh"

namespace gsp {
template gsp_status engine_launch_f16<WeightVal, RedSum>(const EngineLaunch &, const EngineParams &, const WeightVal &,
                                                         cudaStream_t);
template gsp_status engine_launch_f16<WeightOne, RedSum>(const EngineLaunch &, const EngineParams &, const WeightOne &,
                                                         cudaStream_t);
}  // namespace gsp
