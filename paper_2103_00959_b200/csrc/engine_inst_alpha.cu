// engine_inst_alpha.cu -- explicit instantiations of the row-gather engine
// (spmm_engine.cuh) for the "alpha" weight / reduce family; split from the
// callers so nvcc compiles the engine variants in parallel.
#define GSP_ENGINE_INSTANTIATE
#include "spmm_engine.cuh"

namespace gsp {
#define GSP_ENGINE_DEFINE(W, R, tu) GSP_ENGINE_DEFINE_##tu(W, R)
#define GSP_ENGINE_DEFINE_alpha(W, R) \
  template gsp_status engine_launch<W, R>(const EngineLaunch &, const EngineParams &, const W &, cudaStream_t);
#define GSP_ENGINE_DEFINE_sum(W, R)
#define GSP_ENGINE_DEFINE_maxmin(W, R)
#define GSP_ENGINE_DEFINE_gat(W, R)
GSP_ENGINE_INSTANCES(GSP_ENGINE_DEFINE)
}  // namespace gsp
