#pragma once

#include <memory>
#include <optional>
#include <string>

#include "config.h"
#include "trace.h"

namespace as {

struct RunOut {
    Trace trace;
    std::optional<std::string> protocol_error;
};

// Runs one serving session set to completion.
//  clock = virtual  : discrete-event run with profile durations (reference-identical trace)
//  clock = lockstep : same event order and timestamps, every decode step / prefill executed
//                     on the B200 through the asb_* seam (token ids recorded)
//  clock = wall     : real time; step / prefill completions come from the device; prefill and
//                     decode co-run on Green Context partitions for partitioned policies
RunOut serve(const RunCfg& cfg);
Trace serve_or_throw(const RunCfg& cfg);

// Replay checker over a recorded trace (test oracle, not product): ordering, controller
// transitions vs recorded TPOT, token conservation, phase order, committed KV prefixes.
struct ReplayReport {
    int mismatches = 0;
    std::vector<std::string> notes;
    std::string json() const;
};
ReplayReport replay(const Trace& tr);

}  // namespace as
