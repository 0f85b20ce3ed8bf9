// parplan_plan_gpu.hpp — drop-in GPU plan() for the reference parplan library.
// Same signature/semantics as parplan::plan (proj/include/parplan/optimizer.hpp:74-75)
// plus the first CUDA device ordinal and the number of GPUs (devices device ..
// device + n_gpus - 1 of this process; the result is identical for any n_gpus).
#pragma once

#include "parplan/optimizer.hpp"

namespace parplan_gpu {

parplan::PlanResult plan(const parplan::ModelGraph& model, const parplan::Cluster& cluster,
                         const parplan::ProfileTable& profile, int gbs,
                         const parplan::PlanOptions& options = {}, int device = 0, int n_gpus = 1);

}  // namespace parplan_gpu
