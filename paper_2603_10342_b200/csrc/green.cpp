// Green Context slot manager (H1 in SURVEY §2.3) behind asb_slots_*.
//
// Replaces SlotSet (/root/reference/proj/src/executor.hpp:20-42, executor.cpp:9-41):
// the paper pre-establishes one SM partition per reservation level at start-up and rebinds
// the decode / prefill threads between them at run time (§3.3, "<50 us per
// rebinding").  Here every level 1..levels-1 owns a (decode, prefill) pair of green
// contexts built with cuDevSmResourceSplitByCount (decode gets >= level*granularity SMs,
// rounded to the sm_100 split granularity of 8; prefill gets the remainder), each with a
// non-blocking stream.  Level == levels is the full-device shared pair (primary-context
// streams) used by the unpartitioned policies.  Rebind = hand out another pair of streams;
// nothing is created or destroyed on the serving path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "../../include/agentserve_b200.h"

namespace asb {
extern thread_local std::string g_err;
}

namespace {

using FnGetDevResource = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using FnSplit = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                             unsigned int, unsigned int);
using FnGenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
using FnCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
using FnDestroy = CUresult (*)(CUgreenCtx);
using FnStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
using FnStreamDestroy = CUresult (*)(CUstream);

template <typename T>
T entry(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<T>(p);
}

struct Pair {
    CUgreenCtx gd = nullptr, gp = nullptr;
    cudaStream_t sd = nullptr, sp = nullptr;
    int dsms = 0, psms = 0;
};

}  // namespace

struct asb_slots {
    int device = 0;
    int levels = 0;
    int total_sms = 0;
    bool green = false;
    std::vector<Pair> pairs;  // index = level - 1
    FnDestroy destroy = nullptr;
    FnStreamDestroy sdestroy = nullptr;

    ~asb_slots() {
        cudaSetDevice(device);
        for (auto& p : pairs) {
            if (p.gd) {
                if (sdestroy) {
                    sdestroy(reinterpret_cast<CUstream>(p.sd));
                    sdestroy(reinterpret_cast<CUstream>(p.sp));
                }
                if (destroy) {
                    destroy(p.gd);
                    destroy(p.gp);
                }
            } else {
                if (p.sd) cudaStreamDestroy(p.sd);
                if (p.sp && p.sp != p.sd) cudaStreamDestroy(p.sp);
            }
        }
    }
};

extern "C" {

asb_status asb_slots_create(int device, int levels, int granularity_sms, asb_slots** out) {
    if (!out || levels < 2) {
        asb::g_err = "asb_slots_create: need levels >= 2";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    auto fail = [](const std::string& m) {
        asb::g_err = m;
        return ASB_ERR_CUDA;
    };
    if (cudaSetDevice(device) != cudaSuccess) return fail("cudaSetDevice failed");
    cudaFree(nullptr);  // make sure the primary context is active
    auto s = std::make_unique<asb_slots>();
    s->device = device;
    s->levels = levels;
    cudaDeviceGetAttribute(&s->total_sms, cudaDevAttrMultiProcessorCount, device);
    auto get_res = entry<FnGetDevResource>("cuDeviceGetDevResource");
    auto split = entry<FnSplit>("cuDevSmResourceSplitByCount");
    auto gen = entry<FnGenDesc>("cuDevResourceGenerateDesc");
    auto create = entry<FnCreate>("cuGreenCtxCreate");
    auto mkstream = entry<FnStream>("cuGreenCtxStreamCreate");
    s->destroy = entry<FnDestroy>("cuGreenCtxDestroy");
    s->sdestroy = entry<FnStreamDestroy>("cuStreamDestroy_v2");
    if (!s->sdestroy) s->sdestroy = entry<FnStreamDestroy>("cuStreamDestroy");
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    const bool have = get_res && split && gen && create && mkstream && s->destroy && s->sdestroy;
    if (granularity_sms <= 0) granularity_sms = s->total_sms / levels;
    s->pairs.resize(levels);
    bool ok = have;
    for (int lvl = 1; lvl < levels && ok; ++lvl) {
        Pair& p = s->pairs[lvl - 1];
        unsigned want = static_cast<unsigned>(std::max(8, ((lvl * granularity_sms + 7) / 8) * 8));
        want = std::min<unsigned>(want, static_cast<unsigned>(s->total_sms - 8));
        CUdevResource all{}, dec{}, rest{};
        unsigned n = 1;
        if (get_res(static_cast<CUdevice>(device), &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
            split(&dec, &n, &all, &rest, 0, want) != CUDA_SUCCESS || n != 1) {
            ok = false;
            break;
        }
        CUdevResourceDesc dd = nullptr, pd = nullptr;
        if (gen(&dd, &dec, 1) != CUDA_SUCCESS || gen(&pd, &rest, 1) != CUDA_SUCCESS ||
            create(&p.gd, dd, static_cast<CUdevice>(device), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
            create(&p.gp, pd, static_cast<CUdevice>(device), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
            ok = false;
            break;
        }
        CUstream a = nullptr, b = nullptr;
        // decode partition gets the high-priority stream
        if (mkstream(&a, p.gd, CU_STREAM_NON_BLOCKING, hi_prio) != CUDA_SUCCESS ||
            mkstream(&b, p.gp, CU_STREAM_NON_BLOCKING, lo_prio) != CUDA_SUCCESS) {
            ok = false;
            break;
        }
        p.sd = reinterpret_cast<cudaStream_t>(a);
        p.sp = reinterpret_cast<cudaStream_t>(b);
        p.dsms = static_cast<int>(dec.sm.smCount);
        p.psms = static_cast<int>(rest.sm.smCount);
    }
    if (!ok) {
        // No green-context support: destroy what was built and fall back to priority
        // streams on the full device (reported through asb_slots_green() == 0).
        for (auto& p : s->pairs) {
            if (p.sd) s->sdestroy(reinterpret_cast<CUstream>(p.sd));
            if (p.sp) s->sdestroy(reinterpret_cast<CUstream>(p.sp));
            if (p.gd) s->destroy(p.gd);
            if (p.gp) s->destroy(p.gp);
            p = Pair{};
        }
    }
    s->green = ok;
    // shared / fallback streams on the primary context
    for (int lvl = 1; lvl <= levels; ++lvl) {
        Pair& p = s->pairs[lvl - 1];
        if (p.sd) continue;
        if (cudaStreamCreateWithPriority(&p.sd, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
            cudaStreamCreateWithPriority(&p.sp, cudaStreamNonBlocking, lo_prio) != cudaSuccess)
            return fail("cudaStreamCreateWithPriority failed");
        p.dsms = p.psms = s->total_sms;
    }
    *out = s.release();
    return ASB_OK;
}

void asb_slots_free(asb_slots* s) { delete s; }

int asb_slots_levels(const asb_slots* s) { return s ? s->levels : 0; }

int asb_slots_green(const asb_slots* s) { return s && s->green ? 1 : 0; }

asb_status asb_slots_bind(asb_slots* s, int level, void** decode_stream, void** prefill_stream) {
    if (!s || level < 1 || level > s->levels) {
        asb::g_err = "asb_slots_bind: level not in menu";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    const Pair& p = s->pairs[level - 1];
    if (decode_stream) *decode_stream = p.sd;
    if (prefill_stream) *prefill_stream = p.sp;
    return ASB_OK;
}

asb_status asb_slots_sm_counts(const asb_slots* s, int level, int* dsms, int* psms) {
    if (!s || level < 1 || level > s->levels) {
        asb::g_err = "asb_slots_sm_counts: level not in menu";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    if (dsms) *dsms = s->pairs[level - 1].dsms;
    if (psms) *psms = s->pairs[level - 1].psms;
    return ASB_OK;
}

}  // extern "C"
