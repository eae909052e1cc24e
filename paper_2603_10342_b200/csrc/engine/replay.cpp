// Replay checker: recomputes, from the raw events of a recorded trace, the quantities the
// engine recorded and reports every disagreement (role of /root/reference/proj/src/
// replay.cpp:87-335).  Clock-independent checks only, so wall-clock device traces pass:
// event ordering, per-interval ΔL/ΔK and TPOT, controller transitions replayed from the
// recorded TPOT, token conservation, phase order, committed KV prefixes.
#include <cmath>
#include <map>

#include "config.h"
#include "engine.h"

namespace as {

using nlohmann::json;

std::string ReplayReport::json() const {
    nlohmann::json j;
    j["mismatches"] = mismatches;
    j["notes"] = notes;
    return j.dump(2) + "\n";
}

namespace {
bool close(double a, double b) { return std::fabs(a - b) <= 1e-6 * (1.0 + std::fabs(a) + std::fabs(b)); }
}  // namespace

ReplayReport replay(const Trace& tr) {
    ReplayReport r;
    auto bad = [&](const std::string& m) {
        r.mismatches += 1;
        if (r.notes.size() < 200) r.notes.push_back(m);
    };
    RunCfg cfg = config_from_json(tr.config);
    const Policy pol = policy_from(tr.policy);
    const bool adaptive = pol == Policy::AgentServe || pol == Policy::AgentServeNoSlots;

    // 1. ordering
    for (size_t i = 1; i < tr.events.size(); ++i) {
        if (tr.events[i].seq <= tr.events[i - 1].seq) bad("event seq not increasing at " + std::to_string(i));
        if (tr.events[i].t + 1e-9 < tr.events[i - 1].t) bad("event time decreases at seq " + std::to_string(tr.events[i].seq));
    }

    // 2. interval ledger + controller replay
    Ctrl c;
    c.b = cfg.ctrl.b0;
    c.r = cfg.ctrl.r0;
    double dl = 0.0;
    int64_t dk = 0;
    for (const auto& e : tr.events) {
        if (e.kind == Ev::StepDone && e.batch > 0) {
            dl += e.t - e.anchor;
            dk += 1;
        } else if (e.kind == Ev::Tick) {
            const Interval& s = e.sum;
            if (!close(s.dl, dl)) bad("interval " + std::to_string(s.idx) + ": recorded dL " + std::to_string(s.dl) + " != " + std::to_string(dl));
            if (s.dk != dk) bad("interval " + std::to_string(s.idx) + ": recorded dK " + std::to_string(s.dk) + " != " + std::to_string(dk));
            const double tp = dk > 0 ? dl / static_cast<double>(dk) : -1.0;
            if (!close(s.tpot, tp)) bad("interval " + std::to_string(s.idx) + ": TPOT mismatch");
            if (adaptive && s.dk > 0) c = ctrl_step(c, s.tpot, cfg.ctrl);
            if (s.b != c.b || s.r != c.r)
                bad("interval " + std::to_string(s.idx) + ": controller state (" + std::to_string(s.b) + "," +
                    std::to_string(s.r) + ") != replayed (" + std::to_string(c.b) + "," + std::to_string(c.r) + ")");
            dl = 0.0;
            dk = 0;
        }
    }

    // 3-5. per-session: phase order, conservation, committed prefixes
    const size_t n = tr.sessions.size();
    std::vector<std::vector<ReqKind>> order(n);
    std::vector<int> emitted(n, 0), prefix(n, 0), stream_tokens(n, 0);
    for (const auto& e : tr.events) {
        if (e.kind == Ev::Issue && e.s < n) {
            order[e.s].push_back(e.req);
        } else if (e.kind == Ev::StepDone) {
            for (uint32_t s : e.emit)
                if (s < n) emitted[s] += 1;
            if (!e.ids.empty() && e.ids.size() != e.emit.size()) bad("step ids / emit size mismatch");
        } else if (e.kind == Ev::StreamDone && e.s < n) {
            prefix[e.s] += e.tokens;
            stream_tokens[e.s] += e.tokens;
        } else if (e.kind == Ev::PrefillDone && e.s < n) {
            prefix[e.s] += e.len;
            if (e.prefix != prefix[e.s])
                bad("session " + std::to_string(e.s) + ": committed prefix " + std::to_string(e.prefix) +
                    " != recomputed " + std::to_string(prefix[e.s]));
        }
    }
    for (size_t i = 0; i < n; ++i) {
        const SessRec& s = tr.sessions[i];
        const auto& o = order[i];
        bool ok = !o.empty() && o.front() == ReqKind::Cold;
        for (size_t k = 1; ok && k < o.size(); ++k) {
            const ReqKind want = (k % 2 == 1) ? ReqKind::Decode : ReqKind::Resume;
            ok = o[k] == want;
        }
        if (s.done) ok = ok && !o.empty() && o.back() == ReqKind::Decode &&
                         static_cast<int>(o.size()) == 2 + 2 * s.rounds;
        if (!ok) bad("session " + std::to_string(i) + ": phase order violated");
        if (s.done) {
            int want = 0;
            for (int d : s.decodes) want += d;
            if (emitted[i] != want)
                bad("session " + std::to_string(i) + ": emitted " + std::to_string(emitted[i]) + " != planned " + std::to_string(want));
            if (stream_tokens[i] != want) bad("session " + std::to_string(i) + ": stream tokens mismatch");
        }
    }
    return r;
}

}  // namespace as
