// Host-side core: profile curves, workload plans, session FSM, controller, slot menu,
// prefix registry.  Behaviour cited per function against /root/reference/proj/src.
#include "core.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

#include "json.hpp"

namespace as {

using nlohmann::json;

// =================================================================== profile
const char* phase_label(PhaseKind p) {
    switch (p) {
    case PhaseKind::Decode: return "decode";
    case PhaseKind::Cold: return "cold_prefill";
    case PhaseKind::Resume: return "resume_prefill";
    }
    return "?";
}

// On-grid lookup only; 0 SMs -> 0 tokens/s (profile.cpp:24-39).
double Curve::at(int sms, int g) const {
    if (sms == 0) return 0.0;
    const std::string who = phase_label(phase);
    if (sms < g || sms > total_sms)
        raise(Err::Invalid, who + ": allocation " + std::to_string(sms) + " SMs outside grid [" +
                                std::to_string(g) + ", " + std::to_string(total_sms) + "]");
    if (sms % g)
        raise(Err::Invalid, who + ": allocation " + std::to_string(sms) +
                                " SMs is not a multiple of the slot step " + std::to_string(g));
    return pts[static_cast<size_t>(sms / g - 1)].second;
}

static void check_curve(const Curve& c, int g, int S) {
    const std::string who = phase_label(c.phase);
    if (c.total_sms != S)
        raise(Err::Validation, who + ": total_sms " + std::to_string(c.total_sms) +
                                   " differs from bundle total_sms " + std::to_string(S));
    const size_t want = static_cast<size_t>(S / g);
    if (c.pts.size() != want)
        raise(Err::Validation, who + ": expected " + std::to_string(want) + " grid points, got " +
                                   std::to_string(c.pts.size()) +
                                   " (phases must share the grid {g, 2g, ..., S})");
    for (size_t i = 0; i < c.pts.size(); ++i) {
        const int want_sms = static_cast<int>(i + 1) * g;
        if (c.pts[i].first != want_sms)
            raise(Err::Validation, who + ": grid point " + std::to_string(i) + " has sm_count " +
                                       std::to_string(c.pts[i].first) + ", expected " +
                                       std::to_string(want_sms));
        if (!(c.pts[i].second > 0.0))
            raise(Err::Validation,
                  who + ": rate at sm_count " + std::to_string(want_sms) + " must be > 0");
        if (i > 0 && c.pts[i].second < c.pts[i - 1].second)
            raise(Err::Validation, who + ": rate decreases at sm_count " + std::to_string(want_sms) +
                                       " (" + std::to_string(c.pts[i].second) + " < " +
                                       std::to_string(c.pts[i - 1].second) +
                                       "); rates must be non-decreasing in SMs");
    }
}

void Profile::check() const {
    if (g <= 0) raise(Err::Validation, "granularity must be a positive SM count");
    if (S <= 0 || S % g)
        raise(Err::Validation, "total_sms (" + std::to_string(S) +
                                   ") must be a positive multiple of granularity (" +
                                   std::to_string(g) + ")");
    check_curve(dec, g, S);
    check_curve(cold, g, S);
    check_curve(res, g, S);
}

static Curve curve_from(const json& arr, PhaseKind ph, int S, const std::string& key) {
    if (!arr.is_array())
        raise(Err::Validation, "profile." + key + " must be an array of {sms, tokens_per_second}");
    Curve c;
    c.phase = ph;
    c.total_sms = S;
    for (const auto& it : arr) {
        if (!it.contains("sms") || !it.contains("tokens_per_second"))
            raise(Err::Validation, "profile." + key + ": each point needs fields sms and tokens_per_second");
        c.pts.emplace_back(it.at("sms").get<int>(), it.at("tokens_per_second").get<double>());
    }
    return c;
}

Profile profile_from_text(const std::string& text) {
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::parse_error& e) {
        raise(Err::Validation, std::string("profile document is not valid JSON: ") + e.what());
    }
    try {
        Profile p;
        p.S = doc.at("total_sms").get<int>();
        p.g = doc.at("granularity").get<int>();
        p.dec = curve_from(doc.at("decode"), PhaseKind::Decode, p.S, "decode");
        p.cold = curve_from(doc.at("cold_prefill"), PhaseKind::Cold, p.S, "cold_prefill");
        p.res = curve_from(doc.at("resume_prefill"), PhaseKind::Resume, p.S, "resume_prefill");
        p.check();
        return p;
    } catch (const json::exception& e) {
        raise(Err::Validation, std::string("profile document malformed: ") + e.what());
    }
}

static std::string slurp(const std::string& path, const char* what) {
    std::ifstream in(path);
    if (!in) raise(Err::Io, std::string("cannot open ") + what + " file: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

Profile profile_from_file(const std::string& path) { return profile_from_text(slurp(path, "profile")); }

static json curve_json(const Curve& c) {
    json a = json::array();
    for (const auto& [sms, r] : c.pts) a.push_back({{"sms", sms}, {"tokens_per_second", r}});
    return a;
}

std::string profile_text(const Profile& p) {
    json d;
    d["schema"] = "agentsim-profile-v1";
    d["total_sms"] = p.S;
    d["granularity"] = p.g;
    d["decode"] = curve_json(p.dec);
    d["cold_prefill"] = curve_json(p.cold);
    d["resume_prefill"] = curve_json(p.res);
    return d.dump(2) + "\n";
}

// Piecewise-linear rise to a knee, flat after; rounded to 1e-3 (profile.cpp:200-223).
static Curve knee(PhaseKind ph, int S, int g, double peak, double k) {
    Curve c;
    c.phase = ph;
    c.total_sms = S;
    const int n = S / g;
    for (int i = 1; i <= n; ++i) {
        const double share = static_cast<double>(i) / n;
        const double frac = std::min(share / k, 1.0);
        c.pts.emplace_back(i * g, std::round(peak * frac * 1000.0) / 1000.0);
    }
    return c;
}

Profile profile_from_shape(const ProfileShape& s) {
    if (s.total_sms <= 0 || s.granularity <= 0 || s.total_sms % s.granularity)
        raise(Err::Validation, "profile shape: total_sms must be a positive multiple of granularity");
    for (double k : {s.decode_knee, s.cold_knee, s.resume_knee})
        if (!(k > 0.0 && k <= 1.0)) raise(Err::Validation, "profile shape: knees must lie in (0, 1]");
    if (!(s.decode_max_rate > 0.0 && s.cold_max_rate > 0.0 && s.resume_max_rate > 0.0))
        raise(Err::Validation, "profile shape: max rates must be > 0");
    Profile p;
    p.S = s.total_sms;
    p.g = s.granularity;
    p.dec = knee(PhaseKind::Decode, p.S, p.g, s.decode_max_rate, s.decode_knee);
    p.cold = knee(PhaseKind::Cold, p.S, p.g, s.cold_max_rate, s.cold_knee);
    p.res = knee(PhaseKind::Resume, p.S, p.g, s.resume_max_rate, s.resume_knee);
    p.check();
    return p;
}

Profile builtin_profile() { return profile_from_shape(ProfileShape{}); }

// =================================================================== workload
void LenRange::check(const std::string& what) const {
    if (lo < 1) raise(Err::Validation, what + ": min_tokens must be >= 1");
    if (!(lo <= mean && mean <= hi))
        raise(Err::Validation, what + ": need min <= mean <= max, got " + std::to_string(lo) +
                                   " <= " + std::to_string(mean) + " <= " + std::to_string(hi));
}

namespace {
// Expected offset of the truncated law P(k) ~ q^k, k in [0, span]; q > 1 via mirroring.
double law_mean(double q, int span) {
    if (std::fabs(q - 1.0) < 1e-12) return span / 2.0;
    if (q > 1.0) return span - law_mean(1.0 / q, span);
    double num = 0.0, den = 0.0, w = 1.0;
    for (int k = 0; k <= span; ++k) {
        num += k * w;
        den += w;
        w *= q;
    }
    return num / den;
}

double fit_ratio(double target, int span) {
    double lo = 1e-9, hi = 1.0;
    if (target > span / 2.0) {
        lo = 1.0;
        hi = 1.0;
        while (law_mean(hi, span) < target && hi < 1e12) hi *= 2.0;
    }
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        (law_mean(mid, span) < target ? lo : hi) = mid;
    }
    return 0.5 * (lo + hi);
}
}  // namespace

LenLaw::LenLaw(const LenRange& r) : r_(r) {
    r_.check("token distribution");
    const int span = r_.hi - r_.lo;
    if (span == 0) return;
    const double target = static_cast<double>(r_.mean - r_.lo);
    const double q = target <= 0.0 ? 1e-9 : target >= span ? 1e12 : fit_ratio(target, span);
    cdf_.resize(static_cast<size_t>(span) + 1);
    double acc = 0.0, w = 1.0;
    for (int k = 0; k <= span; ++k) {
        acc += w;
        cdf_[static_cast<size_t>(k)] = acc;
        if (q > 1.0 && w > 1e280) {
            for (int j = 0; j <= k; ++j) cdf_[static_cast<size_t>(j)] /= w;
            acc /= w;
            w = 1.0;
        }
        w *= q;
    }
    for (double& c : cdf_) c /= acc;
}

int LenLaw::draw(Stream64& rng) const {
    if (cdf_.empty()) return r_.lo;
    const double u = rng.unit();
    size_t k = static_cast<size_t>(std::lower_bound(cdf_.begin(), cdf_.end(), u) - cdf_.begin());
    if (k >= cdf_.size()) k = cdf_.size() - 1;
    return r_.lo + static_cast<int>(k);
}

void Paradigm::check() const {
    cold.check(name + ".cold");
    resume.check(name + ".resume");
    decode.check(name + ".decode");
    if (rounds < 1) raise(Err::Validation, name + ": steps_per_session must be >= 1");
    if (tool.uniform && !(tool.lo <= tool.hi && tool.lo >= 0.0))
        raise(Err::Validation, name + ": tool_delay uniform range invalid");
    if (!tool.uniform && tool.ms < 0.0) raise(Err::Validation, name + ": tool_delay must be >= 0");
}

// Paper token tables (ToolBench ReAct / Plan-and-Execute; workload.cpp:143-180).
Paradigm paradigm_table(const std::string& paradigm, const std::string& model) {
    struct Row {
        const char* model;
        LenRange react, pe;
    };
    static const Row rows[] = {
        {"qwen2.5-3b", {27, 99, 37}, {41, 125, 55}},
        {"qwen2.5-7b", {21, 127, 45}, {33, 141, 62}},
        {"llama3-8b", {32, 101, 38}, {22, 116, 64}},
    };
    Paradigm p;
    p.cold = LenRange{2500, 3500, 3000};
    if (paradigm != "react" && paradigm != "plan_and_execute")
        raise(Err::Validation, "unknown paradigm '" + paradigm + "' (expected react or plan_and_execute)");
    const bool react = paradigm == "react";
    p.name = paradigm;
    p.resume = react ? LenRange{30, 127, 56} : LenRange{125, 421, 251};
    p.rounds = react ? 4 : 2;
    const Row* hit = nullptr;
    for (const auto& r : rows)
        if (model == r.model) hit = &r;
    if (!hit)
        raise(Err::Validation, "unknown model '" + model + "' (expected qwen2.5-3b, qwen2.5-7b, or llama3-8b)");
    p.decode = react ? hit->react : hit->pe;
    return p;
}

const char* req_label(ReqKind k) {
    switch (k) {
    case ReqKind::Cold: return "cold";
    case ReqKind::Resume: return "resume";
    case ReqKind::Decode: return "decode";
    }
    return "?";
}

const char* stage_label(Stage s) {
    switch (s) {
    case Stage::WaitCold: return "awaiting_cold_prefill";
    case Stage::Decoding: return "decoding";
    case Stage::WaitTool: return "awaiting_tool";
    case Stage::WaitResume: return "awaiting_resume_prefill";
    case Stage::Done: return "done";
    }
    return "?";
}

Paradigm WorkloadCfg::resolve() const {
    Paradigm p = paradigm_table(paradigm, model);
    if (cold) p.cold = *cold;
    if (resume) p.resume = *resume;
    if (decode) p.decode = *decode;
    if (rounds) p.rounds = *rounds;
    if (tool) p.tool = *tool;
    p.check();
    return p;
}

// Pre-sampled plans; per-session sub-streams make plans independent of concurrency
// (workload.cpp:213-246).
std::vector<Plan> make_plans(const WorkloadCfg& w, uint64_t seed) {
    if (w.concurrency < 1) raise(Err::Validation, "workload.concurrency must be >= 1");
    if (w.stagger_ms < 0.0) raise(Err::Validation, "workload.stagger_ms must be >= 0");
    const Paradigm par = w.resolve();
    const LenLaw cold(par.cold), res(par.resume), dec(par.decode);
    std::vector<Plan> out;
    out.reserve(static_cast<size_t>(w.concurrency));
    Stream64 arrivals = Stream64::named(seed, "stagger");
    for (int i = 0; i < w.concurrency; ++i) {
        Plan p;
        p.id = static_cast<uint32_t>(i);
        p.rounds = par.rounds;
        p.arrival = arrivals.between(0.0, w.stagger_ms);
        Stream64 r = Stream64::named(seed, "workload/session/" + std::to_string(i));
        p.cold = cold.draw(r);
        for (int k = 0; k <= par.rounds; ++k) p.decodes.push_back(dec.draw(r));
        for (int k = 0; k < par.rounds; ++k) {
            p.resumes.push_back(res.draw(r));
            p.tools.push_back(par.tool.draw(r));
        }
        p.gid = p.id;
        out.push_back(std::move(p));
    }
    if (w.shard_count > 1) {
        std::vector<Plan> mine;
        for (auto& p : out)
            if (static_cast<int>(p.gid % static_cast<uint32_t>(w.shard_count)) == w.shard_index) {
                p.id = static_cast<uint32_t>(mine.size());
                mine.push_back(std::move(p));
            }
        out = std::move(mine);
    }
    return out;
}

uint64_t plans_hash(const std::vector<Plan>& plans) {
    uint64_t h = Stream64::kFnvOffset;
    auto put = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xff;
            h *= Stream64::kFnvPrime;
        }
    };
    auto putd = [&](double d) {
        uint64_t b;
        std::memcpy(&b, &d, 8);
        put(b);
    };
    for (const auto& p : plans) {
        put(p.id);
        putd(p.arrival);
        put(static_cast<uint64_t>(p.cold));
        put(static_cast<uint64_t>(p.rounds));
        for (int v : p.decodes) put(static_cast<uint64_t>(v));
        for (int v : p.resumes) put(static_cast<uint64_t>(v));
        for (double v : p.tools) putd(v);
    }
    return h;
}

[[noreturn]] static void bad_event(const Plan& p, Done d) {
    raise(Err::Protocol, "session " + std::to_string(p.id) + " in phase " + stage_label(p.stage) +
                             " received mismatched completion event kind " +
                             std::to_string(static_cast<int>(d)));
}

std::optional<Request> advance(Plan& p, Done what, double t, int emitted) {
    switch (p.stage) {
    case Stage::WaitCold:
        if (what != Done::Cold) bad_event(p, what);
        p.cached = p.cold;
        p.stage = Stage::Decoding;
        return Request{p.id, ReqKind::Decode, p.decodes[0], t};
    case Stage::Decoding:
        if (what != Done::Stream) bad_event(p, what);
        p.cached += emitted;
        p.decodes_done += 1;
        p.stage = p.decodes_done > p.rounds ? Stage::Done : Stage::WaitTool;
        return std::nullopt;
    case Stage::WaitTool: {
        if (what != Done::Tool) bad_event(p, what);
        p.stage = Stage::WaitResume;
        const int round = p.decodes_done - 1;
        return Request{p.id, ReqKind::Resume, p.resumes[static_cast<size_t>(round)], t};
    }
    case Stage::WaitResume: {
        if (what != Done::Resume) bad_event(p, what);
        const int round = p.decodes_done - 1;
        p.cached += p.resumes[static_cast<size_t>(round)];
        p.stage = Stage::Decoding;
        return Request{p.id, ReqKind::Decode, p.decodes[static_cast<size_t>(p.decodes_done)], t};
    }
    case Stage::Done:
        bad_event(p, what);
    }
    return std::nullopt;
}

double tool_ms(const Plan& p, int round) {
    if (round < 0 || round >= p.rounds)
        raise(Err::Protocol, "tool delay requested for out-of-range round " + std::to_string(round));
    return p.tools[static_cast<size_t>(round)];
}

// =================================================================== scheduler
Policy policy_from(const std::string& s) {
    if (s == "agentserve") return Policy::AgentServe;
    if (s == "mixed_fcfs") return Policy::MixedFcfs;
    if (s == "static_partition") return Policy::StaticPartition;
    if (s == "chunked_prefill") return Policy::ChunkedPrefill;
    if (s == "agentserve_no_slots") return Policy::AgentServeNoSlots;
    raise(Err::Validation, "unknown policy '" + s +
                               "' (expected agentserve, mixed_fcfs, static_partition, "
                               "chunked_prefill, or agentserve_no_slots)");
}

const char* policy_label(Policy p) {
    switch (p) {
    case Policy::AgentServe: return "agentserve";
    case Policy::MixedFcfs: return "mixed_fcfs";
    case Policy::StaticPartition: return "static_partition";
    case Policy::ChunkedPrefill: return "chunked_prefill";
    case Policy::AgentServeNoSlots: return "agentserve_no_slots";
    }
    return "?";
}

void CtrlCfg::check() const {
    if (!(theta_low > 0.0 && theta_low < theta_high))
        raise(Err::Validation, "controller: need 0 < theta_low < theta_high, got [" +
                                   std::to_string(theta_low) + ", " + std::to_string(theta_high) + "]");
    if (dt <= 0.0) raise(Err::Validation, "controller: delta_t must be > 0");
    if (d_r < 1 || d_b < 1) raise(Err::Validation, "controller: delta_r and delta_b must be >= 1");
    if (b_min < 0 || !(b_min <= b0 && b0 <= b_max))
        raise(Err::Validation, "controller: need 0 <= b_min <= initial_b <= b_max");
    if (r_base < 1)
        raise(Err::Validation, "controller: r_base must be >= 1 slot (decode reservation cannot be empty)");
    if (!(r_base <= r0 && r0 <= total_slots))
        raise(Err::Validation, "controller: need r_base <= initial_r <= total_slots");
}

// Step-level TPOT = ΔL / ΔK, resetting the interval accumulators (scheduler.cpp:55-63).
std::optional<double> take_tpot(Ctrl& c) {
    std::optional<double> v;
    if (c.dk > 0) v = c.dl / static_cast<double>(c.dk);
    c.dl = 0.0;
    c.dk = 0;
    return v;
}

// Algorithm 1 feedback with strict dead band and saturating clamps (scheduler.cpp:65-76).
Ctrl ctrl_step(const Ctrl& c, double tpot, const CtrlCfg& k) {
    Ctrl n = c;
    if (tpot > k.theta_high) {
        n.b = std::max(k.b_min, c.b - k.d_b);
        n.r = std::min(k.total_slots, c.r + k.d_r);
    } else if (tpot < k.theta_low) {
        n.b = std::min(k.b_max, c.b + k.d_b);
        n.r = std::max(k.r_base, c.r - k.d_r);
    }
    return n;
}

// Decode -> QD; resume merges under the budget; cold always QP (scheduler.cpp:78-90).
Queue route(const Request& r, int budget) {
    switch (r.kind) {
    case ReqKind::Decode: return Queue::QD;
    case ReqKind::Resume: return r.len <= budget ? Queue::QD : Queue::QP;
    case ReqKind::Cold: return Queue::QP;
    }
    return Queue::QP;
}

Split partition(Policy p, int static_slots, const Ctrl& c, const CtrlCfg& k) {
    Split s;
    s.budget = c.b;
    switch (p) {
    case Policy::AgentServe:
        s.dslots = c.r;
        s.pslots = k.total_slots - c.r;
        break;
    case Policy::StaticPartition: {
        const int d = static_slots > 0 ? static_slots : k.total_slots / 2;
        s.dslots = d;
        s.pslots = k.total_slots - d;
        break;
    }
    default:
        s.dslots = s.pslots = k.total_slots;
        s.shared = true;
        break;
    }
    if (s.dslots < 1)
        raise(Err::Validation, std::string(policy_label(p)) + ": decode partition would be empty");
    return s;
}

Slots::Slots(int total, double overhead) : total_(total), dec_(1), oh_(overhead) {
    if (total_ < 2) raise(Err::Validation, "slot set needs at least 2 levels");
    if (oh_ < 0.0) raise(Err::Validation, "rebind overhead must be >= 0");
}

int Slots::nearest_above(double target) const {
    if (target > static_cast<double>(total_))
        raise(Err::Infeasible, "reservation target " + std::to_string(target) +
                                   " slots exceeds the device (" + std::to_string(total_) + " slots)");
    return std::max(static_cast<int>(std::ceil(target - 1e-12)), 1);
}

std::optional<Rebind> Slots::bind(int level, double now) {
    if (level < 1 || level > total_)
        raise(Err::Invalid, "rebind level " + std::to_string(level) + " not in menu");
    if (level == dec_) return std::nullopt;
    Rebind r{now, dec_, level, oh_};
    dec_ = level;
    return r;
}

bool Prefixes::sealed(uint32_t s) const {
    auto it = m_.find(s);
    return it != m_.end() && it->second.sealed;
}
int Prefixes::prefix(uint32_t s) const {
    auto it = m_.find(s);
    return it == m_.end() ? 0 : it->second.prefix;
}
void Prefixes::open(uint32_t s) { m_[s].sealed = false; }
void Prefixes::seal_at(uint32_t s, int np) {
    E& e = m_[s];
    if (np < e.prefix)
        raise(Err::Protocol, "kv commit shrinks session " + std::to_string(s) + " prefix from " +
                                 std::to_string(e.prefix) + " to " + std::to_string(np));
    e.prefix = np;
    e.sealed = true;
}
void Prefixes::grow(uint32_t s, int n) {
    E& e = m_[s];
    if (!e.sealed)
        raise(Err::Protocol, "decode append on unsealed KV entry for session " + std::to_string(s));
    e.prefix += n;
}
void Prefixes::need_sealed(uint32_t s) const {
    if (!sealed(s))
        raise(Err::Protocol, "decode step on unsealed KV entry for session " + std::to_string(s));
}

// Virtual-clock decode step: B tokens at mu_D then the admitted chunk at mu_R
// (executor.cpp:84-97).
double step_ms(const Profile& p, int sms, int batch, int chunk) {
    if (batch < 0 || chunk < 0 || (batch == 0 && chunk == 0))
        raise(Err::Invalid, "decode step needs at least one stream or an admitted chunk");
    double ms = 0.0;
    if (batch > 0) ms += 1000.0 * batch / p.mu_d(sms);
    if (chunk > 0) ms += 1000.0 * chunk / p.mu_r(sms);
    return ms;
}

}  // namespace as
