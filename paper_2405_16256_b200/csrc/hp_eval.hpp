// hp_eval.hpp — winner post-processing (hp_evaluate_plan_full).
#pragma once

#include "../../include/hetplan_b200.h"
#include "hp_device.hpp"
#include "hp_host.hpp"

namespace hpe {

hph::Status evaluate_plan_full(hpd::Arena& a, const hph::Problem& p, const hp_plan& plan, hp_plan_eval* eval,
                               hp_stage_eval* stages, hp_trace_event* trace, uint64_t trace_cap);

}  // namespace hpe
