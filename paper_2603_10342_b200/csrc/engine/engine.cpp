// The serving engine: AgentServe's phase-aware scheduler driving the B200 forward.
//
// Request flow, queues, continuous-batching decode steps, Q_P prefill jobs, control ticks
// and the interval ledger follow the reference event loop (/root/reference/proj/src/
// engine.cpp:117-734) so that clock=virtual reproduces its trace byte for byte.  The two
// places where the reference invents time are executed for real when a backend is set:
//   decode step  (reference: start_step -> decode_step_duration_ms, engine.cpp:295-339)
//   prefill unit (reference: start_prefill_unit -> remaining / rate, engine.cpp:442-477)
// and rebinding (engine.cpp:586-602) switches the decode / prefill lanes between
// pre-created Green Context partitions.
#include "engine.h"

#include <algorithm>
#include <cmath>
#include <deque>
#include <memory>
#include <queue>
#include <thread>

#include "devexec.h"

namespace as {

namespace {

constexpr uint64_t kEventCap = 100'000'000;
constexpr double kTimeCap = 1e10;

enum class Mode { Partitioned, Serial, Interleaved };

Mode mode_of(Policy p) {
    switch (p) {
    case Policy::AgentServe:
    case Policy::StaticPartition: return Mode::Partitioned;
    case Policy::MixedFcfs: return Mode::Serial;
    default: return Mode::Interleaved;
    }
}

bool adaptive(Policy p) { return p == Policy::AgentServe || p == Policy::AgentServeNoSlots; }
bool merges(Policy p) {
    return p == Policy::AgentServe || p == Policy::StaticPartition || p == Policy::AgentServeNoSlots;
}

// Heap entries; ties resolve PrefillDone < StepDone < Tick < ToolDone < Arrival, then FIFO.
enum class Kind : int { PrefillDone = 0, StepDone = 1, Tick = 2, ToolDone = 3, Arrival = 4 };
struct Pending {
    double t;
    int prio;
    uint64_t id;
    Kind kind;
    uint32_t s;
    uint64_t gen;
    int round;
    bool operator>(const Pending& o) const {
        if (t != o.t) return t > o.t;
        if (prio != o.prio) return prio > o.prio;
        return id > o.id;
    }
};

struct Job {  // a Q_P prefill (cold, or resume over budget)
    uint32_t s = 0;
    ReqKind kind = ReqKind::Cold;
    int len = 0;
    double issued = 0.0;
    double done = 0.0;      // processed tokens (fractional in virtual mode)
    double started = -1.0;
    int launched = 0;       // tokens handed to the device (wall mode)
    int round = -1;
    std::vector<Seg> segs;
};

struct Admitted {  // resume merged into decode steps under the budget
    uint32_t s = 0;
    int len = 0, left = 0;
    double issued = 0.0;
    bool started = false;
    int round = -1;
    std::vector<Seg> segs;
};

struct Live {
    uint32_t s = 0;
    int left = 0, emitted = 0;
};

struct Step {
    double start = 0.0, end = 0.0, anchor = 0.0;
    int sms = 0;
    std::vector<uint32_t> who;
    int64_t chunk_s = -1;
    int chunk = 0;
    double chunk_ms = 0.0;
    std::vector<int32_t> emitted_ids;
    double dev_ms = -1.0;
};

struct Span {  // open prefill execution span
    double t0 = 0.0, rate = 0.0;
    int sms = 0;
    bool chunk = false;
    int unit_tokens = 0;  // wall mode: tokens of the unit in flight
};

class Engine {
public:
    explicit Engine(const RunCfg& c)
        : c_(c), prof_(c.profile), mode_(mode_of(c.policy)), ctrl_on_(adaptive(c.policy)),
          merge_on_(merges(c.policy)), slots_(c.profile.slots(), c.exec.rebind_oh),
          clock_(c.backend.present ? c.backend.clock : Clock::Virtual) {}

    RunOut run() {
        setup();
        RunOut out;
        try {
            if (clock_ == Clock::Wall) wall_loop();
            else des_loop();
        } catch (const Error& e) {
            if (e.kind != Err::Protocol) throw;
            out.protocol_error = e.what();
        }
        finish();
        out.trace = std::move(tr_);
        return out;
    }

private:
    bool device() const { return clock_ != Clock::Virtual; }

    // ------------------------------------------------------------------ setup
    void setup() {
        plans_ = make_plans(c_.workload, c_.seed);
        tr_.config = c_.to_json();
        tr_.policy = policy_label(c_.policy);
        tr_.seed = c_.seed;
        tr_.hash = plans_hash(plans_);
        for (const auto& p : plans_) {
            SessRec r;
            r.id = p.id;
            r.arrival = p.arrival;
            r.cold = p.cold;
            r.rounds = p.rounds;
            r.decodes = p.decodes;
            r.resumes = p.resumes;
            r.tools = p.tools;
            tr_.sessions.push_back(std::move(r));
        }
        next_tok_.assign(plans_.size(), -1);
        if (device()) dev_ = std::make_unique<DeviceExec>(c_, plans_);
        ctrl_.b = c_.ctrl.b0;
        ctrl_.r = c_.ctrl.r0;
        split_ = partition(c_.policy, c_.static_slots, ctrl_, c_.ctrl);
        if (mode_ == Mode::Partitioned) slots_.bind(split_.dslots, 0.0);  // initial, free
        if (dev_ && clock_ == Clock::Wall) {
            dev_->bind(slots_.decode_level(), split_.shared);
            dev_->clear_rebind_stats();  // the initial binding is set-up, not a rebind
        }
        acct_t0_ = 0.0;
        starved_since_ = 0.0;
        for (const auto& p : plans_) push(p.arrival, Kind::Arrival, p.id);
        push(c_.ctrl.dt, Kind::Tick, 0);
        if (dev_) dev_->start_clock();
    }

    void push(double t, Kind k, uint32_t s, uint64_t gen = 0, int round = 0) {
        heap_.push(Pending{t, static_cast<int>(k), seq_id_++, k, s, gen, round});
    }

    Event ev(Ev k, double t) const {
        Event e;
        e.kind = k;
        e.t = t;
        return e;
    }
    void record(Event e) {
        e.seq = ev_seq_++;
        tr_.events.push_back(std::move(e));
    }

    // ------------------------------------------------------------------ loops
    void des_loop() {
        uint64_t n = 0;
        while (!heap_.empty()) {
            if (n_done_ == plans_.size()) return;
            const Pending p = heap_.top();
            if (c_.horizon && p.t > *c_.horizon) {
                cut(*c_.horizon);
                return;
            }
            heap_.pop();
            if (p.kind == Kind::PrefillDone && p.gen != gen_) continue;  // superseded
            now_ = p.t;
            if (++n > kEventCap || now_ > kTimeCap)
                raise(Err::Protocol, "run exceeded the event or simulated-time guard; "
                                     "likely a starved queue that can never drain");
            dispatch(p);
        }
    }

    void dispatch(const Pending& p) {
        switch (p.kind) {
        case Kind::Arrival: on_arrival(p.s); break;
        case Kind::ToolDone: on_tool(p.s, p.round); break;
        case Kind::PrefillDone: on_prefill_done(); break;
        case Kind::StepDone: on_step_done(); break;
        case Kind::Tick: on_tick(); break;
        }
    }

    // Real time: timers from the heap, completions from the device lanes.
    void wall_loop() {
        uint64_t spins = 0;
        while (n_done_ < plans_.size()) {
            const double t = dev_->now_ms();
            if (c_.horizon && t > *c_.horizon) {
                cut(*c_.horizon);
                return;
            }
            if (stepping_ && dev_->step_ready()) {
                now_ = dev_->now_ms();
                on_step_done();
                continue;
            }
            if (span_ && dev_->prefill_ready()) {
                now_ = dev_->now_ms();
                on_unit_done();
                continue;
            }
            if (!heap_.empty() && heap_.top().t <= t) {
                const Pending p = heap_.top();
                heap_.pop();
                if (p.kind == Kind::Tick && p.gen != tick_gen_) continue;  // superseded by an early tick
                now_ = t;
                dispatch(p);
                continue;
            }
            if (heap_.empty() && !stepping_ && !span_)
                raise(Err::Protocol, "wall-clock run stalled with sessions outstanding");
            if (++spins % 64 == 0) std::this_thread::yield();
        }
    }

    // ------------------------------------------------------------------ requests
    void on_arrival(uint32_t s) {
        Event e = ev(Ev::Arrival, now_);
        e.s = s;
        record(std::move(e));
        issue(Request{s, ReqKind::Cold, plans_[s].cold, now_});
        kick();
    }

    void on_tool(uint32_t s, int round) {
        Event e = ev(Ev::Tool, now_);
        e.s = s;
        e.round = round;
        record(std::move(e));
        auto req = advance(plans_[s], Done::Tool, now_);
        if (!req) raise(Err::Protocol, "tool return produced no resume request");
        issue(*req);
        kick();
    }

    void issue(const Request& r) {
        const int budget = merge_on_ ? ctrl_.b : -1;
        const Queue q = route(r, budget);
        Event e = ev(Ev::Issue, now_);
        e.s = r.session;
        e.req = r.kind;
        e.len = r.len;
        e.q = q;
        e.budget = budget;
        record(std::move(e));
        const int round = plans_[r.session].decodes_done - 1;
        if (q == Queue::QP) {
            Job j;
            j.s = r.session;
            j.kind = r.kind;
            j.len = r.len;
            j.issued = r.t;
            j.round = r.kind == ReqKind::Resume ? round : -1;
            qp_.push_back(std::move(j));
        } else if (r.kind == ReqKind::Decode) {
            waiting_.push_back(r);
            if (!anchored_) {
                anchor_ = std::max(now_, dready_);
                anchored_ = true;
            }
        } else {
            Admitted a;
            a.s = r.session;
            a.len = a.left = r.len;
            a.issued = r.t;
            a.round = round;
            adm_.push_back(std::move(a));
        }
    }

    // ------------------------------------------------------------------ decode side
    int dsms() const { return split_.shared ? prof_.S : prof_.sms_of(slots_.decode_level()); }
    int psms() const { return split_.shared ? prof_.S : prof_.sms_of(slots_.prefill_level()); }
    bool decode_pending() const { return !live_.empty() || !waiting_.empty(); }

    void kv_open(uint32_t s) {
        kv_.open(s);
        if (dev_) dev_->kv_open(s);
    }
    void kv_seal(uint32_t s, int np) {
        kv_.seal_at(s, np);
        if (dev_) dev_->kv_seal(s, np);
    }
    void kv_grow(uint32_t s, int n) {
        kv_.grow(s, n);
        if (dev_) dev_->kv_grow(s, n);
    }
    void kv_need(uint32_t s) {
        kv_.need_sealed(s);
        if (dev_) dev_->kv_need_sealed(s);
    }

    void start_step() {
        while (!waiting_.empty()) {
            const Request& r = waiting_.front();
            kv_need(r.session);
            live_.push_back(Live{r.session, r.len, 0});
            waiting_.pop_front();
        }
        int chunk = 0;
        int64_t chunk_s = -1;
        if (merge_on_ && !adm_.empty()) {
            Admitted& a = adm_.front();
            if (!a.started) {
                a.started = true;
                kv_open(a.s);
            }
            chunk = std::min(c_.exec.resume_chunk, a.left);
            chunk_s = a.s;
        }
        const int batch = static_cast<int>(live_.size());
        if (batch == 0 && chunk == 0) return;
        for (const auto& l : live_) kv_need(l.s);
        const int sms = dsms();
        const double start = std::max(now_, dready_);
        if (!anchored_) {
            anchor_ = start;
            anchored_ = true;
        }
        Step st;
        st.start = start;
        st.anchor = anchor_;
        st.sms = sms;
        for (const auto& l : live_) st.who.push_back(l.s);
        st.chunk_s = chunk_s;
        st.chunk = chunk;
        st.chunk_ms = chunk > 0 ? 1000.0 * chunk / prof_.mu_r(sms) : 0.0;
        if (clock_ == Clock::Wall && mode_ == Mode::Partitioned && c_.backend.lend_idle_prefill)
            dev_->decode_on_full_device(qp_.empty() && !span_);
        if (dev_) launch_step(st);
        if (clock_ == Clock::Wall) {
            st.start = now_;
            st.end = -1.0;
        } else {
            st.end = start + step_ms(prof_, sms, batch, chunk);
        }
        step_ = st;
        stepping_ = true;
        if (clock_ != Clock::Wall) push(step_.end, Kind::StepDone, 0);
        if (clock_ == Clock::Lockstep) collect_step(step_);
    }

    // Build the device batch for a step: one row per live stream (its pending token),
    // plus the admitted-resume chunk rows.
    void launch_step(Step& st) {
        std::vector<DeviceExec::Row> rows;
        rows.reserve(st.who.size());
        for (uint32_t s : st.who) {
            if (next_tok_[s] < 0) raise(Err::Protocol, "stream without a pending token");
            rows.push_back(DeviceExec::Row{s, next_tok_[s]});
            st.emitted_ids.push_back(next_tok_[s]);
        }
        const int32_t* chunk = nullptr;
        bool last = false;
        if (st.chunk > 0) {
            const Admitted& a = adm_.front();
            const auto& toks = dev_->resume_tokens(a.s, a.round);
            chunk = toks.data() + (a.len - a.left);
            last = a.left == st.chunk;
        }
        dev_->step_launch(rows, st.chunk_s, chunk, st.chunk, last);
        chunk_last_ = last;
    }

    void collect_step(Step& st) {
        float ms = -1.f;
        std::vector<int32_t> ids = dev_->step_collect(&ms);
        st.dev_ms = ms;
        for (size_t i = 0; i < st.who.size(); ++i) next_tok_[st.who[i]] = ids[i];
        if (st.chunk > 0 && chunk_last_) next_tok_[static_cast<size_t>(st.chunk_s)] = ids.back();
    }

    void on_step_done() {
        if (clock_ == Clock::Wall) {
            step_.end = now_;
            collect_step(step_);
        }
        Step st = step_;
        stepping_ = false;
        Event e = ev(Ev::StepDone, now_);
        e.step_start = st.start;
        e.anchor = st.anchor;
        e.batch = static_cast<int>(st.who.size());
        e.sms = clock_ == Clock::Wall ? dev_->decode_sms() : st.sms;
        e.emit = st.who;
        e.chunk_s = st.chunk_s;
        e.chunk = st.chunk;
        if (dev_ && c_.backend.emit_ids) e.ids = st.emitted_ids;
        e.dev_ms = st.dev_ms;
        record(std::move(e));
        if (!st.who.empty()) {
            ctrl_.dl += now_ - st.anchor;
            ctrl_.dk += 1;
        }
        if (st.chunk > 0) {
            Admitted& a = adm_.front();
            a.left -= st.chunk;
            acct_res_d_ += st.chunk;
            Seg g;
            g.t0 = clock_ == Clock::Wall ? st.start : now_ - st.chunk_ms;
            g.t1 = now_;
            g.rate = clock_ == Clock::Wall ? (now_ > st.start ? 1000.0 * st.chunk / (now_ - st.start) : 0.0)
                                           : prof_.mu_r(st.sms);
            g.sms = e_sms(st.sms);
            g.tokens = st.chunk;
            g.interval = interval_;
            a.segs.push_back(g);
            if (a.left == 0) {
                Admitted done = std::move(a);
                adm_.pop_front();
                resume_done_in_decode(done);
            }
        }
        std::vector<Live> keep;
        keep.reserve(live_.size());
        for (auto& l : live_) {
            l.left -= 1;
            l.emitted += 1;
            if (l.left > 0) {
                keep.push_back(l);
                continue;
            }
            Event se = ev(Ev::StreamDone, now_);
            se.s = l.s;
            se.tokens = l.emitted;
            record(std::move(se));
            kv_grow(l.s, l.emitted);
            if (advance(plans_[l.s], Done::Stream, now_, l.emitted))
                raise(Err::Protocol, "decode completion emitted a request directly");
            if (plans_[l.s].stage == Stage::Done) {
                finished(l.s);
            } else {
                const int round = plans_[l.s].decodes_done - 1;
                push(now_ + tool_ms(plans_[l.s], round), Kind::ToolDone, l.s, 0, round);
            }
        }
        live_ = std::move(keep);
        if (decode_pending() || (merge_on_ && !adm_.empty())) {
            anchor_ = now_;
        } else {
            anchored_ = false;
        }
        if (mode_ == Mode::Interleaved) last_was_prefill_ = false;
        if (early_tick_due()) {
            tick_gen_ += 1;  // the queued tick of this interval is superseded
            on_tick();       // kicks
            return;
        }
        kick();
    }

    // Controller constants of this tick: backend.theta_high_no_cold_ms replaces theta_high
    // (wall clock) while no cold prefill is queued or running.
    CtrlCfg tick_ctrl() const {
        CtrlCfg k = c_.ctrl;
        const double th = c_.backend.theta_high_no_cold_ms;
        if (clock_ == Clock::Wall && th > k.theta_low &&
            std::none_of(qp_.begin(), qp_.end(), [](const Job& j) { return j.kind == ReqKind::Cold; }))
            k.theta_high = th;
        return k;
    }

    bool early_tick_due() const {
        const int k = c_.backend.early_tick_steps;
        return clock_ == Clock::Wall && k > 0 && ctrl_on_ && mode_ == Mode::Partitioned && ctrl_.dk >= k &&
               ctrl_.dl > c_.ctrl.theta_high * static_cast<double>(ctrl_.dk);
    }

    int e_sms(int sms) const { return clock_ == Clock::Wall ? dev_->decode_sms() : sms; }

    void resume_done_in_decode(Admitted& a) {
        kv_seal(a.s, kv_.prefix(a.s) + a.len);
        Event e = ev(Ev::PrefillDone, now_);
        e.s = a.s;
        e.req = ReqKind::Resume;
        e.len = a.len;
        e.start = a.segs.empty() ? now_ : a.segs.front().t0;
        e.ctx = "decode";
        e.prefix = kv_.prefix(a.s);
        e.segs = a.segs;
        record(std::move(e));
        auto req = advance(plans_[a.s], Done::Resume, now_);
        if (!req) raise(Err::Protocol, "resume completion emitted no decode request");
        issue(*req);
    }

    // ------------------------------------------------------------------ prefill side
    const std::vector<int32_t>& job_tokens(const Job& j) const {
        return j.kind == ReqKind::Cold ? dev_->cold_tokens(j.s) : dev_->resume_tokens(j.s, j.round);
    }

    void start_prefill_unit() {
        if (span_ || qp_.empty()) return;
        if (!split_.shared && split_.pslots == 0) {
            // The partition owns no SMs right now.  Virtual clocks wait (reference semantics).
            // On real kernels a one-row step at R = S/g stays between the controller's
            // thresholds, so R never shrinks and Q_P would starve for ever (livelock seen at
            // C3, 32 agents): run the unit on the stream the lane is bound to (the full device
            // at that level), between decode steps.
            if (clock_ != Clock::Wall || stepping_) return;
        }
        Job& j = qp_.front();
        const int sms = psms();
        const double rate = j.kind == ReqKind::Cold ? prof_.mu_c(sms) : prof_.mu_r(sms);
        const double start = std::max(now_, pready_);
        if (j.started < 0.0) {
            j.started = start;
            if (j.kind == ReqKind::Resume) kv_open(j.s);
        }
        Span sp;
        sp.t0 = start;
        sp.rate = rate;
        sp.sms = sms;
        if (clock_ == Clock::Wall) {
            sp.t0 = now_;
            sp.sms = dev_->prefill_sms();
            sp.chunk = mode_ == Mode::Interleaved;
            const int cap = mode_ == Mode::Interleaved ? std::min(c_.exec.prefill_chunk, dev_->unit_tokens())
                                                       : dev_->unit_tokens();
            const int n = std::min(cap, j.len - j.launched);
            const bool last = j.launched + n == j.len;
            dev_->prefill_launch(j.s, job_tokens(j).data() + j.launched, n, last);
            j.launched += n;
            sp.unit_tokens = n;
            span_ = sp;
            if (mode_ == Mode::Interleaved) last_was_prefill_ = true;
            return;
        }
        const double left = static_cast<double>(j.len) - j.done;
        if (mode_ == Mode::Interleaved) {
            const int chunk = std::min(c_.exec.prefill_chunk, std::max(1, static_cast<int>(std::lround(left))));
            sp.chunk = true;
            push(start + 1000.0 * chunk / rate, Kind::PrefillDone, j.s, gen_);
            last_was_prefill_ = true;
        } else {
            push(start + 1000.0 * left / rate, Kind::PrefillDone, j.s, gen_);
        }
        span_ = sp;
    }

    // Credit the open span up to t to the current interval (virtual clocks only: in wall
    // mode units are credited when they complete).
    void close_span(double t) {
        if (clock_ == Clock::Wall) return;
        if (!span_ || t <= span_->t0) return;
        Job& j = qp_.front();
        Seg g;
        g.t0 = span_->t0;
        g.t1 = t;
        g.rate = span_->rate;
        g.sms = span_->sms;
        g.tokens = span_->rate * (t - span_->t0) / 1000.0;
        g.interval = interval_;
        j.done += g.tokens;
        j.segs.push_back(g);
        credit(j.kind, g.tokens, t - span_->t0);
        span_->t0 = t;
    }

    void credit(ReqKind k, double tokens, double busy) {
        if (k == ReqKind::Cold) {
            acct_cold_ += tokens;
            acct_cold_busy_ += busy;
        } else {
            acct_res_p_ += tokens;
            acct_res_busy_ += busy;
        }
    }

    // wall mode: one launch unit of the head Q_P job finished
    void on_unit_done() {
        Job& j = qp_.front();
        float ms = -1.f;
        const int32_t id = dev_->prefill_collect(&ms);
        Seg g;
        g.t0 = span_->t0;
        g.t1 = now_;
        g.tokens = span_->unit_tokens;
        g.rate = now_ > g.t0 ? 1000.0 * g.tokens / (now_ - g.t0) : 0.0;
        g.sms = span_->sms;
        g.interval = interval_;
        j.done += g.tokens;
        j.segs.push_back(g);
        credit(j.kind, g.tokens, now_ - g.t0);
        j_dev_ms_ += ms;
        const bool chunk_unit = span_->chunk;
        span_.reset();
        if (j.launched < j.len) {
            if (chunk_unit) {
                kick();  // interleave a decode step before the next chunk
            } else {
                start_prefill_unit();
                update_starvation();
            }
            return;
        }
        next_tok_[j.s] = id;
        complete_job(ms);
    }

    void on_prefill_done() {
        if (!span_) raise(Err::Protocol, "prefill completion with no open execution span");
        const bool chunk_unit = span_->chunk;
        close_span(now_);
        span_.reset();
        Job& j = qp_.front();
        bool complete = true;
        if (chunk_unit) {
            complete = j.done >= static_cast<double>(j.len) - 1e-9;
        } else {
            j.done = j.len;
        }
        if (complete) {
            float ms = -1.f;
            if (clock_ == Clock::Lockstep) ms = run_job_now(j);
            complete_job(ms);
        } else {
            kick();
        }
    }

    // lockstep: execute the whole job on the device now, unit by unit
    float run_job_now(Job& j) {
        const auto& toks = job_tokens(j);
        float total = 0.f;
        int32_t id = -1;
        for (int off = 0; off < j.len; off += dev_->unit_tokens()) {
            const int n = std::min(dev_->unit_tokens(), j.len - off);
            const bool last = off + n == j.len;
            dev_->prefill_launch(j.s, toks.data() + off, n, last);
            float ms = 0.f;
            const int32_t r = dev_->prefill_collect(&ms);
            total += ms;
            if (last) id = r;
        }
        next_tok_[j.s] = id;
        return total;
    }

    void complete_job(float ms) {
        Job done = std::move(qp_.front());
        qp_.pop_front();
        kv_seal(done.s, kv_.prefix(done.s) + done.len);
        Event e = ev(Ev::PrefillDone, now_);
        e.s = done.s;
        e.req = done.kind;
        e.len = done.len;
        e.start = done.started;
        e.ctx = mode_ == Mode::Partitioned ? "prefill" : "shared";
        e.prefix = kv_.prefix(done.s);
        e.segs = done.segs;
        if (dev_) {
            e.first_id = next_tok_[done.s];
            e.dev_ms = clock_ == Clock::Wall ? j_dev_ms_ : ms;
        }
        j_dev_ms_ = 0.0;
        record(std::move(e));
        auto req = advance(plans_[done.s], done.kind == ReqKind::Cold ? Done::Cold : Done::Resume, now_);
        if (!req) raise(Err::Protocol, "prefill completion emitted no decode request");
        issue(*req);
        kick();
    }

    // ------------------------------------------------------------------ control
    void on_tick() {
        const double t = now_;
        close_span(t);
        Interval s;
        s.idx = interval_;
        s.t0 = acct_t0_;
        s.t1 = t;
        s.dl = ctrl_.dl;
        s.dk = ctrl_.dk;
        s.dslots = split_.dslots;
        s.pslots = split_.pslots;
        s.shared = split_.shared;
        s.cold_tok = acct_cold_;
        s.res_tok_p = acct_res_p_;
        s.res_tok_d = acct_res_d_;
        s.cold_busy = acct_cold_busy_;
        s.res_busy = acct_res_busy_;
        s.rebind_oh = acct_rebind_;
        flush_starvation(t);
        s.starved = acct_starved_;
        const auto tpot = take_tpot(ctrl_);
        s.tpot = tpot.value_or(-1.0);
        if (ctrl_on_ && tpot) ctrl_ = ctrl_step(ctrl_, *tpot, tick_ctrl());
        s.b = ctrl_.b;
        s.r = ctrl_.r;
        Event te = ev(Ev::Tick, t);
        te.sum = s;
        record(std::move(te));
        interval_ += 1;
        reset_acct(t);
        const Split next = partition(c_.policy, c_.static_slots, ctrl_, c_.ctrl);
        if (mode_ == Mode::Partitioned && next.dslots != slots_.decode_level()) {
            if (auto rb = slots_.bind(next.dslots, t)) {
                double oh = rb->oh;
                if (clock_ == Clock::Wall) oh = dev_->bind(next.dslots, false);  // measured switch cost
                Event e = ev(Ev::Rebind, t);
                e.from = rb->from;
                e.to = rb->to;
                e.oh = oh;
                record(std::move(e));
                acct_rebind_ += oh;
                dready_ = std::max(dready_, t + oh);
                pready_ = std::max(pready_, t + oh);
                if (span_ && clock_ != Clock::Wall) {
                    span_.reset();  // in-flight job resumes after the pause at the new rate
                    gen_ += 1;
                }
            }
        }
        split_ = next;
        if (clock_ == Clock::Wall && c_.backend.early_tick_steps > 0)
            push(now_ + c_.ctrl.dt, Kind::Tick, 0, tick_gen_);  // intervals restart at early ticks
        else
            push(static_cast<double>(interval_ + 1) * c_.ctrl.dt, Kind::Tick, 0);
        kick();
    }

    // ------------------------------------------------------------------ dispatch
    void kick() {
        switch (mode_) {
        case Mode::Partitioned:
            start_prefill_unit();
            if (!stepping_) start_step();
            break;
        case Mode::Serial:
            if (!stepping_ && !span_) {
                if (!qp_.empty()) start_prefill_unit();
                else start_step();
            }
            break;
        case Mode::Interleaved:
            if (!stepping_ && !span_) {
                const bool can_chunk = !qp_.empty();
                const bool can_step = !waiting_.empty() || !live_.empty() || (merge_on_ && !adm_.empty());
                if (can_chunk && can_step) {
                    if (last_was_prefill_) start_step();
                    else start_prefill_unit();
                } else if (can_chunk) {
                    start_prefill_unit();
                } else if (can_step) {
                    start_step();
                }
            }
            break;
        }
        update_starvation();
    }

    void update_starvation() {
        const bool starving = !span_ && qp_.empty();
        if (starving && !starved_since_) {
            starved_since_ = now_;
        } else if (!starving && starved_since_) {
            acct_starved_ += now_ - std::max(*starved_since_, acct_t0_);
            starved_since_.reset();
        }
    }

    void flush_starvation(double t) {
        if (starved_since_) {
            acct_starved_ += t - std::max(*starved_since_, acct_t0_);
            starved_since_ = t;
        }
    }

    void reset_acct(double t0) {
        acct_t0_ = t0;
        acct_cold_ = acct_res_p_ = acct_res_d_ = 0.0;
        acct_cold_busy_ = acct_res_busy_ = 0.0;
        acct_starved_ = 0.0;
        acct_rebind_ = 0.0;
    }

    void finished(uint32_t s) {
        tr_.sessions[s].done = true;
        tr_.sessions[s].done_ms = now_;
        n_done_ += 1;
        if (dev_) dev_->kv_release(s);
    }

    void cut(double h) {
        now_ = h;
        tr_.truncated = true;
        for (auto& r : tr_.sessions)
            if (!r.done) r.truncated = true;
    }

    void finish() {
        close_span(now_);
        flush_starvation(now_);
        tr_.end = now_;
        if (span_ && !qp_.empty()) {
            const Job& j = qp_.front();
            Event e = ev(Ev::PrefillDone, now_);
            e.s = j.s;
            e.req = j.kind;
            e.len = j.len;
            e.start = j.started;
            e.ctx = mode_ == Mode::Partitioned ? "prefill" : "shared";
            e.prefix = -1;
            e.segs = j.segs;
            tr_.inflight = std::move(e);
        }
        if (now_ > acct_t0_) {
            Interval s;
            s.idx = interval_;
            s.t0 = acct_t0_;
            s.t1 = now_;
            s.dl = ctrl_.dl;
            s.dk = ctrl_.dk;
            s.tpot = ctrl_.dk > 0 ? ctrl_.dl / static_cast<double>(ctrl_.dk) : -1.0;
            s.b = ctrl_.b;
            s.r = ctrl_.r;
            s.dslots = split_.dslots;
            s.pslots = split_.pslots;
            s.shared = split_.shared;
            s.cold_tok = acct_cold_;
            s.res_tok_p = acct_res_p_;
            s.res_tok_d = acct_res_d_;
            s.cold_busy = acct_cold_busy_;
            s.res_busy = acct_res_busy_;
            s.starved = acct_starved_;
            s.rebind_oh = acct_rebind_;
            s.partial = true;
            tr_.partial = s;
        }
        if (dev_) {
            if (stepping_ && clock_ == Clock::Wall) dev_->step_collect(nullptr);
            if (span_ && clock_ == Clock::Wall) dev_->prefill_collect(nullptr);
            nlohmann::json d = dev_->describe();
            d["clock"] = clock_ == Clock::Wall ? "wall" : "lockstep";
            tr_.device = d;
        }
    }

    // ------------------------------------------------------------------ state
    const RunCfg& c_;
    const Profile& prof_;
    Mode mode_;
    bool ctrl_on_, merge_on_;
    uint64_t tick_gen_ = 0;  // generation of the queued controller tick (early ticks supersede it)
    Slots slots_;
    Clock clock_;
    std::unique_ptr<DeviceExec> dev_;

    double now_ = 0.0;
    uint64_t seq_id_ = 0, ev_seq_ = 0;
    std::priority_queue<Pending, std::vector<Pending>, std::greater<Pending>> heap_;

    Trace tr_;
    std::vector<Plan> plans_;
    size_t n_done_ = 0;
    std::vector<int32_t> next_tok_;

    std::deque<Job> qp_;
    std::deque<Request> waiting_;
    std::deque<Admitted> adm_;
    std::vector<Live> live_;

    bool stepping_ = false;
    Step step_;
    bool chunk_last_ = false;
    double dready_ = 0.0, anchor_ = 0.0;
    bool anchored_ = false;

    std::optional<Span> span_;
    uint64_t gen_ = 0;
    double pready_ = 0.0;
    double j_dev_ms_ = 0.0;
    std::optional<double> starved_since_;
    bool last_was_prefill_ = false;

    Prefixes kv_;
    Ctrl ctrl_;
    Split split_;
    int interval_ = 0;

    double acct_t0_ = 0.0, acct_cold_ = 0.0, acct_res_p_ = 0.0, acct_res_d_ = 0.0;
    double acct_cold_busy_ = 0.0, acct_res_busy_ = 0.0, acct_starved_ = 0.0, acct_rebind_ = 0.0;
};

}  // namespace

RunOut serve(const RunCfg& cfg) {
    Engine e(cfg);
    return e.run();
}

Trace serve_or_throw(const RunCfg& cfg) {
    RunOut r = serve(cfg);
    if (r.protocol_error) raise(Err::Protocol, *r.protocol_error);
    return std::move(r.trace);
}

}  // namespace as
