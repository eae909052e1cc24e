// Run configuration: one JSON document -> fully resolved config (defaults derived from the
// profile), with the reference's schema (/root/reference/proj/src/config.cpp:54-209) plus an
// optional "backend" section selecting the device executor.
#pragma once

#include <cstdint>
#include <optional>
#include <string>

#include "core.h"
#include "json.hpp"

namespace as {

enum class TpotStat { P95, P50, Mean };
TpotStat tpot_stat_from(const std::string& s);
const char* tpot_stat_label(TpotStat s);

struct Slo {
    double tau_ttft = 0.0, tau_tpot = 0.0, factor = 1.0;
    TpotStat stat = TpotStat::P95;
};

// Thresholds from isolated full-device performance x factor (metrics.cpp:30-43).
Slo calibrate(const Profile& p, double factor, int mean_cold);
double rmin_rate(double tau_tpot_ms);
int rg_star(const Profile& p, double r_min_tps);

struct ExecCfg {
    int total_slots = 0;
    double rebind_oh = 0.05;
    int resume_chunk = 16;
    int prefill_chunk = 256;
};

// Device executor selection (new section; absent => pure virtual-clock run, identical
// to the reference simulator).
enum class Clock { Virtual, Lockstep, Wall };
struct BackendCfg {
    Clock clock = Clock::Virtual;
    std::string model = "tiny";
    uint64_t weight_seed = 0;       // 0: use the run seed
    int device = 0;
    int kv_blocks = 0;              // 0: sized from the workload
    int max_context = 0;            // 0: sized from the workload
    int prefill_unit_tokens = 2048; // launch unit of a Q_P job (rebind granularity)
    bool green_contexts = true;     // Partitioned policies: SM partitions via green contexts
    int green_granularity = 0;      // SMs per slot on the device; 0: device_sms / total_slots
    bool emit_ids = true;           // record generated token ids in the trace
    bool profile_kernels = false;   // per-category kernel timing (CUDA events) in the footer
    // Partitioned policies, wall clock: a decode step launched while Q_P holds no work runs on
    // the full device instead of the decode partition (the idle prefill SMs are lent, and
    // taken back at the next step once prefill work exists)
    bool lend_idle_prefill = false;
    // Adaptive policies, wall clock: close the control interval early once it holds this many
    // decode steps whose mean TPOT already exceeds theta_high (the same Algorithm 1 decision,
    // taken as soon as the evidence is in; the next interval starts then).  0: fixed intervals.
    int early_tick_steps = 0;
    // Adaptive policies, wall clock: theta_high used while Q_P holds no cold prefill (only
    // resume prefills, or none), when prefill SMs cost little TTFT; the controller's
    // theta_high applies during cold bursts.  0: the controller's theta_high throughout.
    double theta_high_no_cold_ms = 0.0;
    bool present = false;
    nlohmann::json to_json() const;
};

struct RunCfg {
    Profile profile;
    WorkloadCfg workload;
    CtrlCfg ctrl;
    ExecCfg exec;
    Slo slo;
    Policy policy = Policy::AgentServe;
    int static_slots = 0;
    std::optional<double> horizon;
    uint64_t seed = 0;
    double r_min_tps = 0.0;
    int rg = 0;
    int mean_cold = 0;
    BackendCfg backend;

    nlohmann::json to_json() const;
};

RunCfg config_from_json(const nlohmann::json& doc);
RunCfg config_from_text(const std::string& text);
RunCfg config_from_file(const std::string& path);

}  // namespace as
