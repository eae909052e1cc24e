#include "devexec.h"

#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace as {

using nlohmann::json;

struct Resident {
    std::string key;
    int ctx = 0, nblocks = 0, dtok = 0, dseg = 0, ptok = 0;
    asb_model* model = nullptr;
    asb_kv* kv = nullptr;
    asb_lane* dlane = nullptr;
    asb_lane* plane = nullptr;
    asb_slots* slots = nullptr;
    int levels = 0;
    bool busy = false;
    ~Resident() {
        if (dlane) asb_lane_free(dlane);
        if (plane) asb_lane_free(plane);
        if (slots) asb_slots_free(slots);
        if (kv) asb_kv_free(kv);
        if (model) asb_model_free(model);
    }
};

namespace {
std::mutex g_res_mu;
std::shared_ptr<Resident> g_res;
}  // namespace

void DeviceExec::ok(asb_status st, const char* what) const {
    if (st == ASB_OK) return;
    const std::string msg = std::string(what) + ": " + asb_last_error();
    if (st == ASB_ERR_PROTOCOL) raise(Err::Protocol, msg);
    if (st == ASB_ERR_INFEASIBLE) raise(Err::Infeasible, msg);
    if (st == ASB_ERR_VALIDATION) raise(Err::Validation, msg);
    raise(Err::Invalid, msg);
}

DeviceExec::DeviceExec(const RunCfg& cfg, const std::vector<Plan>& plans) {
    const BackendCfg& be = cfg.backend;
    unit_ = be.prefill_unit_tokens;
    const uint64_t wseed = be.weight_seed ? be.weight_seed : cfg.seed;
    // longest session context and total KV footprint, from the pre-sampled plans
    int max_ctx = 0;
    int64_t blocks = 0;
    const int bt = asb_kv_block_tokens();
    for (const auto& p : plans) {
        int total = p.cold;
        for (int d : p.decodes) total += d;
        for (int r : p.resumes) total += r;
        max_ctx = std::max(max_ctx, total + 1);
        blocks += (total + bt - 1) / bt + 1;
    }
    const int ctx = be.max_context > 0 ? be.max_context : ((max_ctx + 255) / 256) * 256;
    const int nblocks = be.kv_blocks > 0 ? be.kv_blocks : static_cast<int>(blocks + 8);
    const int n = static_cast<int>(plans.size());
    const int dtok = n + cfg.exec.resume_chunk + 8, dseg = n + 2, ptok = std::max(unit_, 512);
    const int levels = cfg.profile.slots();
    const bool want_slots = be.clock == Clock::Wall && be.green_contexts;
    const std::string key = be.model + "|" + std::to_string(wseed) + "|" + std::to_string(be.device) +
                            "|" + std::to_string(want_slots) + "|" + std::to_string(levels) + "|" +
                            std::to_string(be.green_granularity);
    const bool cache_on = std::getenv("AGENTSERVE_NO_CACHE") == nullptr;
    {
        std::lock_guard<std::mutex> lk(g_res_mu);
        if (cache_on && g_res && !g_res->busy && g_res->key == key && g_res->ctx >= ctx &&
            g_res->nblocks >= nblocks && g_res->dtok >= dtok && g_res->dseg >= dseg && g_res->ptok >= ptok) {
            res_ = g_res;
            res_->busy = true;
        }
    }
    if (!res_) {
        auto r = std::make_shared<Resident>();
        r->key = key;
        r->ctx = ctx;
        r->nblocks = nblocks;
        r->dtok = dtok;
        r->dseg = dseg;
        r->ptok = ptok;
        {
            // drop an idle cached engine first so two models never coexist needlessly
            std::lock_guard<std::mutex> lk(g_res_mu);
            if (g_res && !g_res->busy) g_res.reset();
        }
        ok(asb_model_create(be.model.c_str(), wseed, be.device, ctx, &r->model), "asb_model_create");
        ok(asb_kv_create(r->model, nblocks, &r->kv), "asb_kv_create");
        ok(asb_lane_create(r->model, dtok, dseg, nullptr, &r->dlane), "decode lane");
        ok(asb_lane_create(r->model, ptok, 4, nullptr, &r->plane), "prefill lane");
        if (want_slots) {
            ok(asb_slots_create(be.device, levels, be.green_granularity, &r->slots), "asb_slots_create");
            r->levels = levels;
        }
        r->busy = true;
        res_ = r;
        if (cache_on) {
            std::lock_guard<std::mutex> lk(g_res_mu);
            if (!g_res || !g_res->busy) g_res = r;
        }
    }
    // From here on the resident is marked busy: any throw before the constructor completes
    // (the destructor does not run then) must hand it back, or it would stay pinned forever.
    struct BusyGuard {
        std::shared_ptr<Resident> r;
        bool armed = true;
        ~BusyGuard() {
            if (!armed || !r) return;
            if (r->dlane) asb_lane_wait(r->dlane);
            if (r->plane) asb_lane_wait(r->plane);
            std::lock_guard<std::mutex> lk(g_res_mu);
            r->busy = false;
        }
    } guard{res_};
    model_ = res_->model;
    kv_ = res_->kv;
    dlane_ = res_->dlane;
    plane_ = res_->plane;
    slots_ = res_->slots;
    levels_ = res_->levels;
    char* desc = nullptr;
    ok(asb_model_describe(model_, &desc), "asb_model_describe");
    info_ = json::parse(desc);
    asb_string_free(desc);
    for (const auto& p : plans) sessions_.push_back(p.id);
    for (uint32_t sid : sessions_) asb_kv_release(kv_, sid);  // a reused pool starts empty
    asb_lane_counters(dlane_, nullptr, nullptr, nullptr, 1);
    asb_lane_counters(plane_, nullptr, nullptr, nullptr, 1);
    asb_lane_set_sms(dlane_, 0);
    asb_lane_set_sms(plane_, 0);
    // token streams
    const int V = info_["vocab"].get<int>();
    cold_.resize(plans.size());
    resume_.resize(plans.size());
    for (const auto& p : plans) {
        Stream64 r = Stream64::named(cfg.seed, "tok/" + std::to_string(p.gid) + "/cold");
        auto& c = cold_[p.id];
        c.resize(static_cast<size_t>(p.cold));
        for (auto& t : c) t = static_cast<int32_t>(r.below(static_cast<uint64_t>(V)));
        resume_[p.id].resize(p.resumes.size());
        for (size_t k = 0; k < p.resumes.size(); ++k) {
            Stream64 rr = Stream64::named(cfg.seed, "tok/" + std::to_string(p.gid) + "/resume/" + std::to_string(k));
            auto& v = resume_[p.id][k];
            v.resize(static_cast<size_t>(p.resumes[k]));
            for (auto& t : v) t = static_cast<int32_t>(rr.below(static_cast<uint64_t>(V)));
        }
    }
    if (be.profile_kernels) {
        for (int c = 0; c < ASB_STAT_COUNT; ++c) {  // start from zero
            asb_lane_stats(dlane_, c, nullptr, nullptr, nullptr, 1);
            asb_lane_stats(plane_, c, nullptr, nullptr, nullptr, 1);
        }
        asb_lane_profile(dlane_, 1);
        asb_lane_profile(plane_, 1);
        profiling_ = true;
    }
    info_["kv_blocks"] = res_->nblocks;
    info_["prefill_unit_tokens"] = unit_;
    info_["build"] = asb_build_info();
    start_clock();
    guard.armed = false;
}

DeviceExec::~DeviceExec() {
    if (!res_) return;
    asb_lane_wait(dlane_);
    asb_lane_wait(plane_);
    for (uint32_t sid : sessions_) asb_kv_release(kv_, sid);
    asb_lane_profile(dlane_, 0);
    asb_lane_profile(plane_, 0);
    std::lock_guard<std::mutex> lk(g_res_mu);
    res_->busy = false;
}

void DeviceExec::step_launch(const std::vector<Row>& rows, int64_t chunk_s, const int32_t* chunk,
                             int chunk_n, bool chunk_logits) {
    std::vector<asb_segment> segs;
    std::vector<int32_t> toks;
    segs.reserve(rows.size() + 1);
    for (const auto& r : rows) {
        segs.push_back(asb_segment{r.s, 1, 1});
        toks.push_back(r.tok);
    }
    if (chunk_s >= 0 && chunk_n > 0) {
        segs.push_back(asb_segment{static_cast<uint32_t>(chunk_s), chunk_n, chunk_logits ? 1 : 0});
        toks.insert(toks.end(), chunk, chunk + chunk_n);
    }
    step_logit_rows_ = static_cast<int>(rows.size()) + (chunk_s >= 0 && chunk_n > 0 && chunk_logits ? 1 : 0);
    ok(asb_forward(dlane_, kv_, segs.data(), static_cast<int>(segs.size()), toks.data()), "decode step");
    step_t0_ = now_ms();
    static const bool trace_launch = std::getenv("AGENTSERVE_TRACE_LAUNCHES") != nullptr;
    if (trace_launch)
        std::fprintf(stderr, "[%9.3f] step rows=%zu chunk=%d sms=%d\n", step_t0_, rows.size(), chunk_n, dsms_);
    step_what_ = "decode step (" + std::to_string(rows.size()) + " rows + chunk " + std::to_string(chunk_n) +
                 " on " + std::to_string(dsms_) + " SMs)";
}

// A launch that has not completed after kLaunchTimeoutMs is a device fault: fail the run with
// the launch named instead of spinning forever.
static constexpr double kLaunchTimeoutMs = 10000.0;

bool DeviceExec::step_ready() const {
    if (asb_lane_query(dlane_) == 1) return true;
    if (now_ms() - step_t0_ > kLaunchTimeoutMs) raise(Err::Protocol, step_what_ + " did not complete in 10 s");
    return false;
}

std::vector<int32_t> DeviceExec::step_collect(float* dev_ms) {
    std::vector<int32_t> ids(static_cast<size_t>(std::max(step_logit_rows_, 1)));
    ok(asb_lane_fetch(dlane_, ids.data(), step_logit_rows_, nullptr), "decode fetch");
    ids.resize(static_cast<size_t>(step_logit_rows_));
    if (dev_ms) *dev_ms = asb_lane_last_ms(dlane_);
    return ids;
}

void DeviceExec::prefill_launch(uint32_t s, const int32_t* toks, int n, bool want) {
    asb_segment g{s, n, want ? 1 : 0};
    prefill_want_ = want;
    ok(asb_forward(plane_, kv_, &g, 1, toks), "prefill unit");
    pre_t0_ = now_ms();
    static const bool trace_launch = std::getenv("AGENTSERVE_TRACE_LAUNCHES") != nullptr;
    if (trace_launch)
        std::fprintf(stderr, "[%9.3f] prefill s=%u n=%d len=%d sms=%d\n", pre_t0_, s, n, asb_kv_length(kv_, s), psms_);
    pre_what_ = "prefill unit (" + std::to_string(n) + " tokens of session " + std::to_string(s) + " at length " +
                std::to_string(asb_kv_length(kv_, s)) + " on " + std::to_string(psms_) + " SMs)";
}

bool DeviceExec::prefill_ready() const {
    if (asb_lane_query(plane_) == 1) return true;
    if (now_ms() - pre_t0_ > kLaunchTimeoutMs) raise(Err::Protocol, pre_what_ + " did not complete in 10 s");
    return false;
}

int32_t DeviceExec::prefill_collect(float* dev_ms) {
    int32_t id = -1;
    if (prefill_want_) {
        ok(asb_lane_fetch(plane_, &id, 1, nullptr), "prefill fetch");
    } else {
        ok(asb_lane_wait(plane_), "prefill wait");
    }
    if (dev_ms) *dev_ms = asb_lane_last_ms(plane_);
    return id;
}

double DeviceExec::bind(int level, bool shared) {
    if (!slots_) return 0.0;
    const double t0 = now_ms();
    const int lvl = shared ? levels_ : level;
    void *sd = nullptr, *sp = nullptr;
    ok(asb_slots_bind(slots_, lvl, &sd, &sp), "asb_slots_bind");
    ok(asb_slots_sm_counts(slots_, lvl, &part_dsms_, &psms_), "sm counts");
    level_ = lvl;
    if (dfull_ && lvl != levels_) {
        // keep borrowing the full device; the partition stream is taken at the next step
        // that runs while prefill work exists (decode_on_full_device(false))
    } else {
        ok(asb_lane_set_stream(dlane_, sd), "bind decode lane");
        dsms_ = part_dsms_;
        ok(asb_lane_set_sms(dlane_, green() ? dsms_ : 0), "lane sms");
    }
    ok(asb_lane_set_stream(plane_, sp), "bind prefill lane");
    ok(asb_lane_set_sms(plane_, green() ? psms_ : 0), "lane sms");
    const double ms = now_ms() - t0;
    rebind_us_.push_back(1000.0 * ms);
    return ms;
}

void DeviceExec::decode_on_full_device(bool on) {
    if (!slots_ || !green() || on == dfull_) return;
    void* sd = nullptr;
    const int lvl = on ? levels_ : level_;
    ok(asb_slots_bind(slots_, lvl, &sd, nullptr), "asb_slots_bind");
    int d = 0;
    ok(asb_slots_sm_counts(slots_, lvl, &d, nullptr), "sm counts");
    ok(asb_lane_set_stream(dlane_, sd), "lend decode lane");
    dsms_ = d;
    ok(asb_lane_set_sms(dlane_, lvl == levels_ ? 0 : dsms_), "lane sms");
    dfull_ = on;
    lend_switches_ += 1;
}

bool DeviceExec::green() const { return slots_ && asb_slots_green(slots_) == 1; }

void DeviceExec::kv_open(uint32_t s) { ok(asb_kv_begin_write(kv_, s), "kv begin_write"); }

void DeviceExec::kv_seal(uint32_t s, int np) {
    ok(asb_kv_commit(kv_, s, np), "kv commit");
    const int len = asb_kv_length(kv_, s);
    if (len != np)
        raise(Err::Protocol, "device KV holds " + std::to_string(len) + " tokens for session " +
                                 std::to_string(s) + " at commit of prefix " + std::to_string(np));
}

void DeviceExec::kv_grow(uint32_t s, int n) {
    ok(asb_kv_append(kv_, s, n), "kv append");
    const int len = asb_kv_length(kv_, s), pre = asb_kv_prefix(kv_, s);
    if (len != pre)
        raise(Err::Protocol, "device KV holds " + std::to_string(len) + " tokens for session " +
                                 std::to_string(s) + " but the registry prefix is " + std::to_string(pre));
}

void DeviceExec::kv_need_sealed(uint32_t s) { ok(asb_kv_require_sealed(kv_, s), "kv require_sealed"); }

int DeviceExec::kv_len(uint32_t s) const { return asb_kv_length(kv_, s); }

void DeviceExec::kv_release(uint32_t s) { ok(asb_kv_release(kv_, s), "kv release"); }

json DeviceExec::describe() const {
    json j = info_;
    {
        int64_t l0 = 0, h0 = 0, d0 = 0, l1 = 0, h1 = 0, d1 = 0;
        asb_lane_counters(dlane_, &l0, &h0, &d0, 0);
        asb_lane_counters(plane_, &l1, &h1, &d1, 0);
        j["io"] = {{"kernel_launches", l0 + l1}, {"h2d_bytes", h0 + h1}, {"d2h_bytes", d0 + d1}};
    }
    if (profiling_) {
        static const char* names[ASB_STAT_COUNT] = {"decode_attn", "prefill_attn", "decode_gemm",
                                                     "prefill_gemm", "forward", "decode_step"};
        static const char* units[ASB_STAT_COUNT] = {"bytes", "flops", "bytes", "flops", "tokens", "bytes"};
        json k = json::object();
        for (int c = 0; c < ASB_STAT_COUNT; ++c) {
            json lanes = json::object();
            for (int which = 0; which < 2; ++which) {
                double ms = 0.0, u = 0.0;
                int64_t n = 0;
                asb_lane_stats(which == 0 ? dlane_ : plane_, c, &ms, &u, &n, 0);
                lanes[which == 0 ? "decode_lane" : "prefill_lane"] = {{"ms", ms}, {"units", u}, {"launches", n}};
            }
            lanes["unit"] = units[c];
            k[names[c]] = lanes;
        }
        j["kernels"] = k;
    }
    j["green_contexts"] = green();
    j["levels"] = levels_;
    {
        // rebind latency (host cost of switching both lanes; non-blocking) vs the paper's
        // < 50 us
        std::vector<double> v = rebind_us_;
        std::sort(v.begin(), v.end());
        auto pct = [&](double p) {
            if (v.empty()) return -1.0;
            size_t k = static_cast<size_t>(std::ceil(p / 100.0 * double(v.size())));
            k = std::max<size_t>(1, std::min(k, v.size()));
            return v[k - 1];
        };
        j["rebind_us"] = {{"n", v.size()}, {"p50", pct(50)}, {"p99", pct(99)}, {"max", v.empty() ? -1.0 : v.back()}};
        j["lend_switches"] = lend_switches_;
    }
    if (slots_) {
        json lv = json::array();
        for (int l = 1; l <= levels_; ++l) {
            int d = 0, p = 0;
            asb_slots_sm_counts(slots_, l, &d, &p);
            lv.push_back({{"level", l}, {"decode_sms", d}, {"prefill_sms", p}});
        }
        j["partitions"] = lv;
    }
    return j;
}

}  // namespace as
