// Competitive-ratio verification (restates /root/reference/proj/src/analysis.cpp:160-242).
#pragma once
#include <string>

#include "json.hpp"
#include "trace.h"

namespace as {

struct VerifyResult {
    int checked = 0, vacuous = 0, violations = 0;
    bool assumptions_met = true;
    std::string json;  // agentsim-verify-v1 document, formatted as the reference's
};

// params_doc: {"delta_sms": x, "eps_bar": y}, both optional (default: measured maxima).
VerifyResult verify_trace(const Trace& trace, const nlohmann::json& params_doc);

}  // namespace as
