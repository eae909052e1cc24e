// Append-only run record in the reference's JSONL schema v1
// (/root/reference/proj/src/trace.hpp:63-145, trace.cpp:95-351), so the reference's own
// metrics / replay code can read traces produced by real device runs.  Device runs add
// keys the reference parser ignores: "ids" / "dev_ms" on step_done, "first_id" / "dev_ms"
// on prefill_done, and a "device" object in the footer.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "core.h"
#include "json.hpp"

namespace as {

enum class Ev { Arrival, Issue, PrefillDone, StepDone, StreamDone, Tool, Tick, Rebind };
const char* ev_label(Ev e);

struct Seg {
    double t0 = 0.0, t1 = 0.0, rate = 0.0;
    int sms = 0;
    double tokens = 0.0;
    int interval = 0;
};

struct Interval {
    int idx = 0;
    double t0 = 0.0, t1 = 0.0;
    double dl = 0.0;
    int64_t dk = 0;
    double tpot = -1.0;
    int b = 0, r = 0, dslots = 0, pslots = 0;
    bool shared = false;
    double cold_tok = 0.0, res_tok_p = 0.0, res_tok_d = 0.0;
    double cold_busy = 0.0, res_busy = 0.0, starved = 0.0, rebind_oh = 0.0;
    bool partial = false;
};

struct Event {
    Ev kind = Ev::Arrival;
    double t = 0.0;
    uint64_t seq = 0;
    uint32_t s = 0;
    // issue
    ReqKind req = ReqKind::Cold;
    int len = 0;
    Queue q = Queue::QP;
    int budget = 0;
    // prefill_done
    double start = 0.0;
    std::string ctx;
    int prefix = 0;
    std::vector<Seg> segs;
    // step_done
    double step_start = 0.0, anchor = 0.0;
    int batch = 0, sms = 0;
    std::vector<uint32_t> emit;
    int64_t chunk_s = -1;
    int chunk = 0;
    // stream_done
    int tokens = 0;
    // tool
    int round = -1;
    // tick
    Interval sum;
    // rebind
    int from = 0, to = 0;
    double oh = 0.0;
    // device extras (absent in virtual runs)
    std::vector<int32_t> ids;
    int32_t first_id = -1;
    double dev_ms = -1.0;
};

struct SessRec {
    uint32_t id = 0;
    double arrival = 0.0;
    int cold = 0, rounds = 0;
    std::vector<int> decodes, resumes;
    std::vector<double> tools;
    bool done = false, truncated = false;
    double done_ms = -1.0;
};

struct Trace {
    int schema = 1;
    nlohmann::json config;
    std::string policy;
    uint64_t seed = 0, hash = 0;
    std::vector<SessRec> sessions;
    std::vector<Event> events;
    std::optional<Interval> partial;
    std::optional<Event> inflight;
    double end = 0.0;
    bool truncated = false;
    nlohmann::json device;  // null for virtual runs

    std::vector<Interval> intervals() const;
    std::string jsonl() const;
    static Trace parse(const std::string& text);
    void save(const std::string& path) const;
    static Trace load(const std::string& path);
};

// ------------------------------------------------------------------ metrics
// (/root/reference/proj/src/metrics.cpp:45-214; p99 added for the B200 report)
double nearest_rank(std::vector<double> v, double p);

struct SessMetrics {
    uint32_t id = 0;
    bool completed = false, has_output = false;
    double ttft = -1.0;
    int emitted = 0;
    std::vector<double> gaps;
    double p50 = -1.0, p95 = -1.0, p99 = -1.0, mean = -1.0;
    bool ttft_ok = false, tpot_ok = false, slo_met = false;
};

struct Summary {
    std::vector<SessMetrics> sessions;
    double ttft_p50 = -1.0, ttft_p95 = -1.0, ttft_p99 = -1.0;
    double tpot_p50 = -1.0, tpot_p95 = -1.0, tpot_p99 = -1.0;
    double tps = 0.0;
    double slo = 0.0, slo_ttft = 0.0, slo_tpot = 0.0;
    int completed = 0;
    double tau_ttft = 0.0, tau_tpot = 0.0, factor = 0.0;
    std::string stat;
};

Summary summarize(const Trace& tr, double tau_ttft, double tau_tpot, double factor,
                  const std::string& stat);
std::string summary_json(const Summary& m, const Trace& tr);
std::string summary_csv(const Summary& m, const Trace& tr);

}  // namespace as
