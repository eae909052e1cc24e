// Host-side core of the AgentServe serving engine: error taxonomy, named-substream RNG,
// throughput profiles, workload plans + session state machine, controller / classifier /
// partition decision, slot menu and KV prefix registry.
//
// Semantics follow the reference scheduler library (/root/reference/proj/src) so that a
// virtual-clock run reproduces its trace byte for byte; the code is a B200-side restatement
// organised around the device executor, not a translation.
#pragma once

#include <cstdint>
#include <deque>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace as {

// ------------------------------------------------------------------ errors
// Kinds map 1:1 onto agsv_status (/root/reference/proj/src/error.hpp:10-17).
enum class Err { Invalid, Validation, Protocol, Io, NoData, Infeasible };

struct Error : std::runtime_error {
    Err kind;
    Error(Err k, const std::string& m) : std::runtime_error(m), kind(k) {}
};
[[noreturn]] inline void raise(Err k, const std::string& m) { throw Error(k, m); }

// ------------------------------------------------------------------ RNG
// splitmix64 with FNV-1a-named sub-streams (/root/reference/proj/src/rng.hpp:14-60).
struct Stream64 {
    uint64_t s = 0;
    static constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
    static constexpr uint64_t kFnvPrime = 0x00000100000001b3ull;
    static uint64_t fnv(std::string_view name) {
        uint64_t h = kFnvOffset;
        for (unsigned char c : name) {
            h ^= c;
            h *= kFnvPrime;
        }
        return h;
    }
    static uint64_t finalize(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    static Stream64 named(uint64_t seed, std::string_view name) {
        Stream64 r;
        r.s = finalize(seed ^ fnv(name));
        return r;
    }
    uint64_t u64() {
        s += 0x9e3779b97f4a7c15ull;
        return finalize(s);
    }
    double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
    double between(double lo, double hi) { return lo + (hi - lo) * unit(); }
    uint64_t below(uint64_t n) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(u64()) * n) >> 64);
    }
};

// ------------------------------------------------------------------ profile
enum class PhaseKind { Decode, Cold, Resume };
const char* phase_label(PhaseKind p);

struct Curve {
    PhaseKind phase = PhaseKind::Decode;
    std::vector<std::pair<int, double>> pts;  // (sms, tokens/s) on the grid {g..S}
    int total_sms = 0;
    double at(int sms, int g) const;
};

struct Profile {
    Curve dec, cold, res;
    int g = 0;  // SMs per slot
    int S = 0;  // total SMs
    int slots() const { return S / g; }
    int sms_of(int slots) const { return slots * g; }
    double mu_d(int sms) const { return dec.at(sms, g); }
    double mu_c(int sms) const { return cold.at(sms, g); }
    double mu_r(int sms) const { return res.at(sms, g); }
    void check() const;
};

struct ProfileShape {
    int total_sms = 120;
    int granularity = 12;
    double decode_max_rate = 100.0, decode_knee = 0.2;
    double cold_max_rate = 1500.0, cold_knee = 0.8;
    double resume_max_rate = 800.0, resume_knee = 0.4;
};

Profile profile_from_text(const std::string& text);
Profile profile_from_file(const std::string& path);
std::string profile_text(const Profile& p);
Profile profile_from_shape(const ProfileShape& s);
Profile builtin_profile();

// ------------------------------------------------------------------ workload
struct LenRange {
    int lo = 1, hi = 1, mean = 1;
    void check(const std::string& what) const;
};

// Truncated-geometric length law with support [lo, hi] and expectation `mean`
// (/root/reference/proj/src/workload.cpp:72-118).
class LenLaw {
public:
    explicit LenLaw(const LenRange& r);
    int draw(Stream64& rng) const;

private:
    LenRange r_;
    std::vector<double> cdf_;
};

struct ToolDelay {
    bool uniform = false;
    double ms = 100.0, lo = 0.0, hi = 0.0;
    double draw(Stream64& rng) const { return uniform ? rng.between(lo, hi) : ms; }
};

struct Paradigm {
    std::string name;
    LenRange cold, resume, decode;
    int rounds = 1;
    ToolDelay tool;
    void check() const;
};

Paradigm paradigm_table(const std::string& paradigm, const std::string& model);

enum class ReqKind { Cold, Resume, Decode };
const char* req_label(ReqKind k);

struct Request {
    uint32_t session = 0;
    ReqKind kind = ReqKind::Cold;
    int len = 0;
    double t = 0.0;
};

enum class Stage { WaitCold, Decoding, WaitTool, WaitResume, Done };
const char* stage_label(Stage s);

struct Plan {
    uint32_t id = 0;
    uint32_t gid = 0;  // id in the global (unsharded) workload: names its token streams
    Stage stage = Stage::WaitCold;
    int cached = 0;
    int rounds = 0;
    int decodes_done = 0;
    double arrival = 0.0;
    int cold = 0;
    std::vector<int> decodes;    // rounds + 1
    std::vector<int> resumes;    // rounds
    std::vector<double> tools;   // rounds
};

enum class Done { Cold, Stream, Tool, Resume };

struct WorkloadCfg {
    std::string paradigm = "react";
    std::string model = "qwen2.5-7b";
    int concurrency = 3;
    double stagger_ms = 500.0;
    std::optional<LenRange> cold, resume, decode;
    std::optional<int> rounds;
    std::optional<ToolDelay> tool;
    // replica sharding (multi-GPU): keep sessions with gid % shard_count == shard_index
    int shard_index = 0, shard_count = 1;
    Paradigm resolve() const;
};

std::vector<Plan> make_plans(const WorkloadCfg& w, uint64_t seed);
uint64_t plans_hash(const std::vector<Plan>& plans);
// Session FSM (/root/reference/proj/src/workload.cpp:284-325).
std::optional<Request> advance(Plan& p, Done what, double t, int emitted = 0);
double tool_ms(const Plan& p, int round);

// ------------------------------------------------------------------ scheduler
enum class Policy { AgentServe, MixedFcfs, StaticPartition, ChunkedPrefill, AgentServeNoSlots };
Policy policy_from(const std::string& s);
const char* policy_label(Policy p);

struct CtrlCfg {
    double theta_low = 0.0, theta_high = 0.0;
    int d_r = 1, d_b = 64;
    double dt = 250.0;
    int b_min = 64, b_max = 1024, r_base = 1, b0 = 256, r0 = 1, total_slots = 10;
    void check() const;
};

struct Ctrl {
    int b = 0;           // resume-prefill token budget B_prefill
    int r = 0;           // decode slot floor R_min
    double dl = 0.0;     // ΔL
    int64_t dk = 0;      // ΔK
};

std::optional<double> take_tpot(Ctrl& c);
Ctrl ctrl_step(const Ctrl& c, double tpot, const CtrlCfg& k);

enum class Queue { QD, QP };
Queue route(const Request& r, int budget);

struct Split {
    int dslots = 0, pslots = 0;
    bool shared = false;
    int budget = 0;
};
Split partition(Policy p, int static_slots, const Ctrl& c, const CtrlCfg& k);

struct Rebind {
    double t = 0.0;
    int from = 0, to = 0;
    double oh = 0.0;
};

class Slots {
public:
    Slots(int total, double overhead);
    int total() const { return total_; }
    int decode_level() const { return dec_; }
    int prefill_level() const { return total_ - dec_; }
    int nearest_above(double target) const;
    std::optional<Rebind> bind(int level, double now);

private:
    int total_, dec_;
    double oh_;
};

// Host view of the KV read-only handoff (prefix + seal).  The device pool mirrors it.
class Prefixes {
public:
    bool sealed(uint32_t s) const;
    int prefix(uint32_t s) const;
    void open(uint32_t s);
    void seal_at(uint32_t s, int new_prefix);
    void grow(uint32_t s, int n);
    void need_sealed(uint32_t s) const;

private:
    struct E {
        int prefix = 0;
        bool sealed = false;
    };
    std::map<uint32_t, E> m_;
};

double step_ms(const Profile& p, int sms, int batch, int chunk);

}  // namespace as
