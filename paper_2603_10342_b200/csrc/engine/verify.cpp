// Competitive-ratio verification of an AgentServe trace: restates
// verify_trace and the bound helpers of /root/reference/proj/src/analysis.cpp:13-242 and the
// ProfileBundle helpers of /root/reference/proj/src/profile.cpp:41-77 on the engine's types.
// On a virtual-clock trace the report is identical to the reference's (the interval ledger is
// byte-identical); on a wall-clock B200 trace the ledger holds the prefill tokens the real
// kernels processed per interval, so rho is the measured competitive ratio.
#include <algorithm>
#include <cmath>
#include <optional>
#include <string>
#include <vector>

#include "config.h"
#include "json.hpp"
#include "trace.h"
#include "verify.h"

namespace as {

using nlohmann::json;

namespace {

// ProfileBundle::mixed_prefill_rate (profile.cpp:41-49)
double mixed_rate(const Profile& p, double eta, int sms) {
    if (!(eta >= 0.0 && eta <= 1.0)) raise(Err::Invalid, "eta must lie in [0, 1], got " + std::to_string(eta));
    if (sms == 0) return 0.0;
    return eta * p.mu_c(sms) + (1.0 - eta) * p.mu_r(sms);
}

// ProfileBundle::lipschitz_estimate (profile.cpp:51-69)
double lipschitz(const Profile& p, double eta, int lo, int hi) {
    if (lo > hi)
        raise(Err::Invalid, "lipschitz_estimate: empty window [" + std::to_string(lo) + ", " + std::to_string(hi) + "]");
    mixed_rate(p, eta, lo);
    mixed_rate(p, eta, hi);
    double max_slope = 0.0;
    for (int x = std::max(lo, p.g); x + p.g <= hi; x += p.g) {
        const double d = std::fabs(mixed_rate(p, eta, x + p.g) - mixed_rate(p, eta, x));
        max_slope = std::max(max_slope, d / p.g);
    }
    if (lo == 0 && hi >= p.g) max_slope = std::max(max_slope, mixed_rate(p, eta, p.g) / p.g);
    return max_slope;
}

// ProfileBundle::grid_floor (profile.cpp:71-77)
int grid_floor(const Profile& p, double sms) {
    if (sms < p.g) return 0;
    const int level = static_cast<int>(std::floor(sms / p.g + 1e-12));
    return std::min(level, p.slots()) * p.g;
}

struct Pieces {
    double denom = 0.0;
    int offline = 0, reduced = 0;
    double delta_eff = 0.0;
};

// bound_pieces (analysis.cpp:95-121)
Pieces pieces(const Profile& p, double eta, int rg, double delta_sms, double eps_bar) {
    if (delta_sms < 0.0) raise(Err::Invalid, "delta must be >= 0");
    if (!(eps_bar >= 0.0 && eps_bar < 1.0)) raise(Err::Invalid, "eps_bar must lie in [0, 1)");
    Pieces q;
    q.offline = p.sms_of(p.slots() - rg);
    q.denom = mixed_rate(p, eta, q.offline);
    if (!(q.denom > 0.0)) raise(Err::Infeasible, "degenerate capacity: mu_P(S - R_g*) = 0, bound undefined");
    const double reduced = static_cast<double>(q.offline) - delta_sms;
    if (reduced < 0.0) raise(Err::Invalid, "delta exceeds the offline prefill allocation (S - R_g*)");
    q.reduced = grid_floor(p, reduced);
    q.delta_eff = static_cast<double>(q.offline - q.reduced);
    return q;
}

struct IntervalReport {
    int index = 0;
    double w_a = 0.0, w_star = 0.0, rho = 0.0, bound = 0.0, lin = 0.0, eta = 0.0;
    bool vacuous = false, satisfied = true;
};

}  // namespace

VerifyResult verify_trace(const Trace& tr, const json& params_doc) {
    const RunCfg cfg = config_from_json(tr.config);
    const Profile& p = cfg.profile;
    std::optional<double> p_delta, p_eps;
    if (params_doc.contains("delta_sms")) p_delta = params_doc.at("delta_sms").get<double>();
    if (params_doc.contains("eps_bar")) p_eps = params_doc.at("eps_bar").get<double>();
    const double rel_tol = 1e-9;
    const double dt = cfg.ctrl.dt;

    VerifyResult rep;
    std::vector<IntervalReport> out;
    double min_rho = 0.0, min_bound = 0.0, measured_delta = 0.0, measured_eps = 0.0;
    bool met = true;
    std::vector<std::string> flags;
    const int rg = rg_star(p, cfg.r_min_tps);
    if (tr.policy != "agentserve") {
        met = false;
        flags.push_back("policy is '" + tr.policy + "', bounds apply to agentserve runs");
    }
    if (cfg.ctrl.r_base < rg) {
        met = false;
        flags.push_back("r_base (" + std::to_string(cfg.ctrl.r_base) + " slots) < R_g* (" + std::to_string(rg) +
                        " slots): feasibility floor not configured");
    }
    std::vector<Interval> ivs;
    for (const auto& s : tr.intervals())
        if (!s.partial) ivs.push_back(s);
    for (const auto& s : ivs) {
        const double overshoot = static_cast<double>(s.dslots - rg) * p.g;
        measured_delta = std::max(measured_delta, std::max(0.0, overshoot));
        measured_eps = std::max(measured_eps, s.rebind_oh / dt);
        if (s.dslots < rg) {
            met = false;
            flags.push_back("interval " + std::to_string(s.idx) + ": decode binding below R_g* (feasibility floor violated)");
        }
    }
    const double delta = p_delta.value_or(measured_delta), eps = p_eps.value_or(measured_eps);
    if (p_delta && measured_delta > *p_delta + 1e-9) {
        met = false;
        flags.push_back("measured overshoot " + std::to_string(measured_delta) + " SMs exceeds the stated delta bound");
    }
    if (p_eps && measured_eps > *p_eps + 1e-12) {
        met = false;
        flags.push_back("measured rebind loss exceeds the stated eps bound");
    }
    bool first = true;
    for (const auto& s : ivs) {
        IntervalReport r;
        r.index = s.idx;
        const double busy = s.cold_busy + s.res_busy;
        r.eta = busy > 0.0 ? s.cold_busy / busy : 0.0;
        r.w_a = s.cold_tok + s.res_tok_p + s.res_tok_d;
        // offline_optimum (analysis.cpp:34-47)
        const double w_star = mixed_rate(p, r.eta, p.sms_of(p.slots() - rg)) * dt / 1000.0;
        r.w_star = w_star;
        r.vacuous = (w_star <= 0.0) || (s.starved > 1e-9);
        if (!r.vacuous) {
            r.rho = r.w_a / w_star;
            const Pieces q = pieces(p, r.eta, rg, delta, eps);
            r.bound = (1.0 - eps) * mixed_rate(p, r.eta, q.reduced) / q.denom;          // analysis.cpp:125-130
            r.lin = (1.0 - eps) * (1.0 - lipschitz(p, r.eta, q.reduced, q.offline) * q.delta_eff / q.denom);
            r.satisfied = r.rho >= r.bound - rel_tol * std::max(1.0, std::fabs(r.bound));
            rep.checked += 1;
            if (!r.satisfied) rep.violations += 1;
            if (first || r.rho < min_rho) min_rho = r.rho;
            if (first || r.bound < min_bound) min_bound = r.bound;
            first = false;
        } else {
            rep.vacuous += 1;
        }
        out.push_back(r);
    }
    rep.assumptions_met = met;
    // VerifyReport::to_json (analysis.cpp:134-158)
    json j;
    j["schema"] = "agentsim-verify-v1";
    j["checked"] = rep.checked;
    j["vacuous"] = rep.vacuous;
    j["violations"] = rep.violations;
    j["min_rho"] = min_rho;
    j["min_bound"] = min_bound;
    j["measured_delta_sms"] = measured_delta;
    j["measured_eps"] = measured_eps;
    j["used_delta_sms"] = delta;
    j["used_eps_bar"] = eps;
    j["r_g_star_slots"] = rg;
    j["assumptions_met"] = met;
    j["assumption_flags"] = flags;
    j["intervals"] = json::array();
    for (const auto& r : out)
        j["intervals"].push_back({{"idx", r.index},
                                  {"w_a", r.w_a},
                                  {"w_star", r.w_star},
                                  {"rho", r.rho},
                                  {"bound", r.bound},
                                  {"linearized_bound", r.lin},
                                  {"eta", r.eta},
                                  {"vacuous", r.vacuous},
                                  {"satisfied", r.satisfied}});
    rep.json = j.dump(2) + "\n";
    return rep;
}

}  // namespace as
