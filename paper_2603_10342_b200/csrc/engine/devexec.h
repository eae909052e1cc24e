// Engine-side device executor: owns the asb_* handles (model, paged KV pool, decode and
// prefill lanes, green-context slots) and the synthetic token streams.  The host engine
// talks to CUDA only through this class, which talks only to the asb_* C ABI.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/agentserve_b200.h"
#include "config.h"
#include "json.hpp"

namespace as {

// Device state that outlives one run: weights, KV pool, lanes, green contexts.  Cached
// process-wide so back-to-back agsv_simulate calls with a compatible backend reuse the
// resident model instead of re-initialising it (set AGENTSERVE_NO_CACHE=1 to disable).
struct Resident;

class DeviceExec {
public:
    DeviceExec(const RunCfg& cfg, const std::vector<Plan>& plans);
    ~DeviceExec();
    DeviceExec(const DeviceExec&) = delete;
    DeviceExec& operator=(const DeviceExec&) = delete;

    // wall clock, ms since start_clock()
    void start_clock() { t0_ = std::chrono::steady_clock::now(); }
    double now_ms() const {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    }

    // synthetic prompt / tool-output ids ("tok/<session>/cold", "tok/<session>/resume/<r>")
    const std::vector<int32_t>& cold_tokens(uint32_t s) const { return cold_[s]; }
    const std::vector<int32_t>& resume_tokens(uint32_t s, int round) const { return resume_[s][round]; }

    // ---- decode lane: B single-token rows (+ one admitted-resume chunk)
    struct Row {
        uint32_t s;
        int32_t tok;
    };
    void step_launch(const std::vector<Row>& rows, int64_t chunk_s, const int32_t* chunk, int chunk_n,
                     bool chunk_logits);
    bool step_ready() const;
    // ids for every row (+ chunk id last when chunk_logits); device ms
    std::vector<int32_t> step_collect(float* dev_ms);

    // ---- prefill lane: one launch unit of a Q_P job
    void prefill_launch(uint32_t s, const int32_t* toks, int n, bool want_logits);
    bool prefill_ready() const;
    int32_t prefill_collect(float* dev_ms);  // -1 when the unit produced no logits

    // ---- SM partitions
    // Rebind both lanes to the (decode, prefill) streams of a slot level (shared = the
    // full-device pair).  Non-blocking: in-flight work finishes on its old partition.
    // Returns the measured host cost in ms.
    double bind(int decode_level, bool shared);
    // Work-conserving decode (backend.lend_idle_prefill): while the prefill partition has
    // nothing to run, the decode lane borrows the full device; it returns to its partition
    // at the next step once prefill work exists.  No-op without green contexts.
    void decode_on_full_device(bool on);
    bool decode_borrowing() const { return dfull_; }
    void clear_rebind_stats() { rebind_us_.clear(); }
    bool green() const;
    int decode_sms() const { return dsms_; }
    int prefill_sms() const { return psms_; }

    // ---- KV protocol mirror (the device registry must agree with the host one)
    void kv_open(uint32_t s);
    void kv_seal(uint32_t s, int new_prefix);
    void kv_grow(uint32_t s, int n);
    void kv_need_sealed(uint32_t s);
    int kv_len(uint32_t s) const;
    void kv_release(uint32_t s);

    int unit_tokens() const { return unit_; }
    nlohmann::json describe() const;

private:
    void ok(asb_status st, const char* what) const;

    std::shared_ptr<Resident> res_;
    asb_model* model_ = nullptr;
    asb_kv* kv_ = nullptr;
    asb_lane* dlane_ = nullptr;
    asb_lane* plane_ = nullptr;
    asb_slots* slots_ = nullptr;
    int levels_ = 0;
    std::vector<uint32_t> sessions_;
    int dsms_ = 0, psms_ = 0;
    int level_ = 0, part_dsms_ = 0;  // current slot level and its decode partition size
    bool dfull_ = false;
    int64_t lend_switches_ = 0;
    std::vector<double> rebind_us_;  // measured host cost of every rebind (non-blocking)
    int unit_ = 2048;
    int step_logit_rows_ = 0;
    bool prefill_want_ = false;
    bool profiling_ = false;
    std::vector<std::vector<int32_t>> cold_;
    std::vector<std::vector<std::vector<int32_t>>> resume_;
    std::chrono::steady_clock::time_point t0_;
    double step_t0_ = 0.0, pre_t0_ = 0.0;  // launch times (watchdog)
    std::string step_what_, pre_what_;
    nlohmann::json info_;
};

}  // namespace as
