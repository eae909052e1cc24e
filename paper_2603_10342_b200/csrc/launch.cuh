// Kernel launch helper: every forward-path kernel goes out through cudaLaunchKernelEx so it can
// carry the programmatic-stream-serialization attribute (PDL).  A PDL launch may begin while
// the previous kernel on the stream is still draining; the kernel itself calls pdl_wait()
// (griddepcontrol.wait) before touching anything that kernel wrote, and pdl_trigger() early so
// the next launch overlaps its own tail.  Without the attribute both are no-ops.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace asb {

// Per host thread: whether launches issued now carry the PDL attribute (set by asb_forward
// for the duration of one forward; off while per-launch profiling events are recorded).
inline thread_local bool tl_pdl = false;

// Whether the previous launch on this host thread was a thread-block-cluster launch.  A kernel
// launched programmatically (PDL) right after a cluster launch is launched WITHOUT the attribute:
// its griddepcontrol.wait did not reliably order it after the cluster grid's stores here (the
// decode step was run-to-run nondeterministic when the fused QKV GEMM ran as S-CTA split-K
// clusters; deterministic with the same kernels and no PDL, or with single-CTA tiles:
// scripts/determinism.py, profiles/r2_pdl_cluster_determinism.txt).  ASB_PDL_AFTER_CLUSTER=1
// restores PDL there (A/B only).
inline thread_local bool tl_prev_cluster = false;
inline bool pdl_for_launch(bool is_cluster) {
    static const bool after_cluster = std::getenv("ASB_PDL_AFTER_CLUSTER") &&
                                      std::atoi(std::getenv("ASB_PDL_AFTER_CLUSTER")) != 0;
    const bool use = tl_pdl && (after_cluster || !tl_prev_cluster);
    tl_prev_cluster = is_cluster;
    return use;
}

struct PdlScope {
    bool prev;
    explicit PdlScope(bool on) : prev(tl_pdl) { tl_pdl = on; }
    ~PdlScope() { tl_pdl = prev; }
};

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    if (pdl_for_launch(false)) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace asb
