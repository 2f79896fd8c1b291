// Multi-device scenes: one process, several B200s (include/cvpb200.h,
// "multi-device scenes").
//
// A group is a list of member contexts holding the same scene. The reference
// caller's view list is sharded in contiguous ranges and its volume in
// contiguous z-slabs (k slowest, geometry.hpp:34-36). Each member runs on its
// own host thread (pageable host copies then proceed in parallel) and its own
// stream; members meet at a host barrier only where data crosses devices, and
// the cross-device dependency itself is a CUDA event recorded by the producer
// and waited on by the consumer's stream:
//
//   forward   slab upload (H2D, float64 -> float32)  | barrier |
//             all-gather of the other slabs (peer copies over NVLink), then
//             the member's views -> its part of the host stack
//   backward  fused (CVP, default): | barrier | every member's bricks store
//             their voxels straight into the owning member's receive region
//             for that source over peer memory (cvpb_backproject_cvp_scatter,
//             store mode: the exchange overlaps the bricks still computing)
//             | barrier | each owner sums its regions in member order
//             (cvpb_sum_slabs, float64) -> its slab of the host volume;
//             two-pass (TT / Siddon, no peer access): the
//             member's part of the stack -> a full partial volume | barrier |
//             launch_reduce_slab64 reads the member's slab out of every
//             member's partial over peer memory, sums the members in a fixed
//             order, writes float64 -> its slab of the host volume
//   cgls      the reference's recurrence (solver.cpp:55-106) with x, p, s
//             held as slabs, r, q as view shards, dots summed over members in
//             a fixed order; p is all-gathered before every forward.
//
// Every member computes the same scalars from the same published partials,
// so all members take the same branches (no broadcast is needed). With one
// member the group forwards to the single-context entry points.
#include "cvpb200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels.hpp"

namespace {

constexpr int kAborted = 1000;  // a member stopped because another one failed

#define G_CUDA(call)                                                                              \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return cvpb::set_last_error(                                                          \
                CVPB_CUDA_ERROR, (std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call).c_str()); \
    } while (0)

#define G_TRY(call)                     \
    do {                                \
        int rc_ = (call);               \
        if (rc_ != CVPB_OK) return rc_; \
    } while (0)

int fail(int code, const char* msg) { return cvpb::set_last_error(code, msg); }

template <class T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t reserve(size_t want) {  // on the current device
        if (want <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(want, 1));
        if (e == cudaSuccess) n = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// Host barrier that a failing member can break: wait() then returns false in
// every member and they unwind instead of waiting for a peer that is gone.
class Barrier {
public:
    explicit Barrier(int n) : n_(n) {}
    bool wait() {
        std::unique_lock<std::mutex> l(mu_);
        if (aborted_) return false;
        const long g = gen_;
        if (++waiting_ == n_) {
            waiting_ = 0;
            ++gen_;
            cv_.notify_all();
            return true;
        }
        cv_.wait(l, [&] { return gen_ != g || aborted_; });
        return !aborted_;
    }
    void abort() {
        std::lock_guard<std::mutex> l(mu_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex mu_;
    std::condition_variable cv_;
    int n_, waiting_ = 0;
    long gen_ = 0;
    bool aborted_ = false;
};

#define G_SYNC(bar)                          \
    do {                                     \
        if (!(bar).wait()) return kAborted;  \
    } while (0)

double kahan(const double* v, size_t n) {
    double sum = 0.0, c = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double y = v[i] - c;
        const double t = sum + y;
        c = (t - sum) - y;
        sum = t;
    }
    return sum;
}

}  // namespace

struct cvpb_group {
    struct Member {
        int device = 0;
        cvpb_context* ctx = nullptr;
        cudaStream_t st = nullptr;
        cudaEvent_t ev_ready = nullptr;  // this member's slab / partial is ready for its peers
        cudaEvent_t ev_done = nullptr;   // fused backward: this member's scatter is complete
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        int v0 = 0, nv = 0;     // view shard
        size_t s0 = 0, ns = 0;  // volume slab [elements]
        Buf<float> vol;         // full volume (forward input; CGLS: p, own slab = p's slab)
        Buf<float> part;        // full partial volume (backward)
        Buf<float> proj, q;     // the member's views (CGLS: r, q)
        Buf<float> sx, ss;      // slabs (CGLS: x, s)
        Buf<double> stage;      // float64 staging of host transfers
        Buf<double> partials;   // dot partials
        Buf<float> gather;      // reduce-scatter without peer access: the slabs of every member
        Buf<float> recv;        // fused backward: one slab-sized region per member (its voxels)
        Buf<int> flag;
    };
    std::vector<Member> m;
    bool direct_peer = true;  // every member can load every other member's memory
    bool peer_atomics = true;  // ... and add to it with native atomics (fused reduce-scatter)
    bool has_geometry = false;
    cvpb_volume_geometry vol{};
    cvpb_detector_geometry det{};
    int n_views = 0;
    size_t nvox = 0, npx = 0;
    std::mutex mu;  // one call at a time (members share the group's buffers)
    std::vector<double> pub;  // per-member published scalars (written before a barrier)
};

namespace {

int check_group(cvpb_group* g, bool need_geometry = true) {
    if (!g) return fail(CVPB_INVALID_ARGUMENT, "null group");
    if (need_geometry && !g->has_geometry) return fail(CVPB_INVALID_ARGUMENT, "no geometry set on the group");
    return CVPB_OK;
}

// Run f(member, barrier) on one host thread per member (member 0 on the
// caller's thread). The first real failure is the call's status and message.
template <class F>
int run_members(cvpb_group* g, F&& f) {
    const int n = int(g->m.size());
    Barrier bar(n);
    std::vector<int> rc(n, CVPB_OK);
    std::vector<std::string> msg(n);
    auto body = [&](int i) {
        int r = cudaSetDevice(g->m[i].device) == cudaSuccess
                    ? f(i, bar)
                    : fail(CVPB_CUDA_ERROR, "cannot select a member's device");
        if (r != CVPB_OK) {
            rc[i] = r;
            msg[i] = cvpb_last_error();
            bar.abort();
        }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < n; ++i) th.emplace_back(body, i);
    body(0);
    for (auto& t : th) t.join();
    cudaSetDevice(g->m[0].device);
    for (int i = 0; i < n; ++i)
        if (rc[i] != CVPB_OK && rc[i] != kAborted) return fail(rc[i], msg[i].c_str());
    for (int i = 0; i < n; ++i)
        if (rc[i] != CVPB_OK) return fail(CVPB_RUNTIME_ERROR, "multi-device call aborted");
    return CVPB_OK;
}

// the operator of a call: 0 CVP, 1 Siddon-K, 2 TT (cvpb_cgls numbering)
struct Op {
    int kind = 0;
    cvpb_cvp_options cvp{CVPB_SCALING_EXACT, 1, CVPB_PRECISION_EXACT, CVPB_R_CUT_CENTROID};
    cvpb_tt_options tt{1};
    cvpb_exec_policy exec{0, 0, 0};
    int k = 1;
};

int op_forward(const Op& op, cvpb_group::Member& mb, const float* vol, float* proj) {
    if (mb.nv == 0) return CVPB_OK;
    if (op.kind == 0) return cvpb_project_cvp(mb.ctx, &op.cvp, &op.exec, vol, proj, mb.v0, mb.nv, mb.st);
    if (op.kind == 1)
        return cvpb_project_siddon(mb.ctx, op.k, nullptr, &op.exec, vol, proj, mb.v0, mb.nv, mb.st);
    return cvpb_project_tt(mb.ctx, &op.tt, vol, proj, mb.v0, mb.nv, mb.st);
}

int op_backward(const Op& op, cvpb_group::Member& mb, size_t nvox, const float* proj, float* vol) {
    if (mb.nv == 0) {
        G_CUDA(cudaMemsetAsync(vol, 0, sizeof(float) * nvox, mb.st));
        return CVPB_OK;
    }
    if (op.kind == 0)
        return cvpb_backproject_cvp(mb.ctx, &op.cvp, &op.exec, proj, vol, mb.v0, mb.nv, 0, mb.st);
    if (op.kind == 1)
        return cvpb_backproject_siddon(mb.ctx, op.k, &op.exec, proj, vol, mb.v0, mb.nv, 0, mb.st);
    return cvpb_backproject_tt(mb.ctx, &op.tt, proj, vol, mb.v0, mb.nv, 0, mb.st);
}

// float64 host range -> float32 device (through the member's staging buffer)
int upload(cvpb_group::Member& mb, const double* host, float* dev, size_t n) {
    if (n == 0) return CVPB_OK;
    G_CUDA(cudaMemcpyAsync(mb.stage.p, host, sizeof(double) * n, cudaMemcpyHostToDevice, mb.st));
    G_CUDA(cvpb::launch_f64_to_f32(mb.stage.p, dev, n, mb.st));
    return CVPB_OK;
}

int download(cvpb_group::Member& mb, const float* dev, double* host, size_t n) {
    if (n == 0) return CVPB_OK;
    G_CUDA(cvpb::launch_f32_to_f64(dev, mb.stage.p, n, mb.st));
    G_CUDA(cudaMemcpyAsync(host, mb.stage.p, sizeof(double) * n, cudaMemcpyDeviceToHost, mb.st));
    return CVPB_OK;
}

// all-gather: every other member's slab of its `vol` buffer into ours
int gather_slabs(cvpb_group* g, int i) {
    auto& mb = g->m[i];
    for (size_t h = 0; h < g->m.size(); ++h) {
        auto& o = g->m[h];
        if (int(h) == i || o.ns == 0) continue;
        G_CUDA(cudaStreamWaitEvent(mb.st, o.ev_ready, 0));
        G_CUDA(cudaMemcpyPeerAsync(mb.vol.p + o.s0, mb.device, o.vol.p + o.s0, o.device,
                                   sizeof(float) * o.ns, mb.st));
    }
    return CVPB_OK;
}

// reduce-scatter: this member's slab summed over every member's `part`
// (after their ev_ready), into out32 (float32, device) or out64 (float64, device)
int reduce_slab(cvpb_group* g, int i, float* out32, double* out64) {
    auto& mb = g->m[i];
    if (mb.ns == 0) return CVPB_OK;
    const int n = int(g->m.size());
    cvpb::SlabSources src{};
    for (int h = 0; h < n; ++h) G_CUDA(cudaStreamWaitEvent(mb.st, g->m[h].ev_ready, 0));
    if (g->direct_peer) {
        for (int h = 0; h < n; ++h) src.p[h] = g->m[h].part.p + mb.s0;
    } else {
        // no peer mapping between some members: stage the slabs with peer copies
        G_CUDA(mb.gather.reserve(mb.ns * n));
        for (int h = 0; h < n; ++h) {
            G_CUDA(cudaMemcpyPeerAsync(mb.gather.p + mb.ns * h, mb.device, g->m[h].part.p + mb.s0,
                                       g->m[h].device, sizeof(float) * mb.ns, mb.st));
            src.p[h] = mb.gather.p + mb.ns * h;
        }
    }
    if (out32) G_CUDA(cvpb::launch_reduce_slab(src, n, mb.ns, out32, mb.st));
    if (out64) G_CUDA(cvpb::launch_reduce_slab64(src, n, mb.ns, out64, mb.st));
    return CVPB_OK;
}

// Backward with the reduce-scatter fused in (CVP): every member's bricks
// store their voxels straight into the owning member's receive buffer — one
// slab-sized region per source member, peer memory over NVLink
// (cvpb_backproject_cvp_scatter, store mode) — and each owner then sums its
// regions locally in member order (cvpb_sum_slabs). Plain stores, no
// atomics (a member's launch writes each of its voxels once), and the sum
// order is fixed, so the result is bit-reproducible and deterministic mode is
// served too. Needs peer access between every pair of members;
// CVPB_GROUP_FUSED=0 forces the two-pass path (full partial volumes +
// fixed-order peer-load reduction).
bool fused_backward(const cvpb_group* g, const Op& op) {
    if (op.kind != 0 || !g->direct_peer || !g->peer_atomics) return false;
    const char* e = std::getenv("CVPB_GROUP_FUSED");
    return !(e && e[0] == '0');
}

// Scatter this member's views into every owner's receive region for this
// member, meet, then sum the own receive buffer into out32 / out64 (the
// member's slab). Stream-ordered: on return the sum is enqueued on mb.st.
int scatter_backward(cvpb_group* g, int i, Barrier& bar, const Op& op, const float* proj, float* out32,
                     double* out64) {
    auto& mb = g->m[i];
    const int n = int(g->m.size());
    G_CUDA(mb.recv.reserve(std::max<size_t>(mb.ns * n, 1)));
    // the receive buffers are free (their previous sums are enqueued before)
    G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));
    G_SYNC(bar);
    for (int h = 0; h < n; ++h) G_CUDA(cudaStreamWaitEvent(mb.st, g->m[h].ev_ready, 0));
    cvpb_slab_targets tg{};
    tg.n = n;
    tg.store = 1;
    const size_t plane = size_t(g->vol.counts[0]) * g->vol.counts[1];
    for (int h = 0; h < n; ++h) {
        tg.plane_begin[h] = int(g->m[h].s0 / plane);
        tg.slab[h] = g->m[h].recv.p + size_t(i) * g->m[h].ns;  // owner h's region for source i
    }
    tg.plane_begin[n] = g->vol.counts[2];
    if (mb.nv)
        G_TRY(cvpb_backproject_cvp_scatter(mb.ctx, &op.cvp, &op.exec, proj, mb.v0, mb.nv, &tg, mb.st));
    else
        for (int h = 0; h < n; ++h)  // no views: this source contributes zeros
            if (g->m[h].ns)
                G_CUDA(cudaMemsetAsync(tg.slab[h], 0, sizeof(float) * g->m[h].ns, mb.st));
    G_CUDA(cudaEventRecord(mb.ev_done, mb.st));
    G_SYNC(bar);  // every member's scatter is recorded
    for (int h = 0; h < n; ++h) G_CUDA(cudaStreamWaitEvent(mb.st, g->m[h].ev_done, 0));
    if (mb.ns) {
        std::vector<const float*> src(n);
        for (int h = 0; h < n; ++h) src[h] = mb.recv.p + size_t(h) * mb.ns;
        G_TRY(cvpb_sum_slabs(mb.ctx, src.data(), n, mb.ns, out32, out64, mb.st));
    }
    return CVPB_OK;
}

// compensated float64 dot of two float32 device vectors, synchronous
int dot(cvpb_group::Member& mb, const float* a, const float* b, size_t n, double* out) {
    const int np = cvpb::dot_partials_count();
    std::vector<double> h(np);
    G_CUDA(cvpb::launch_dot(a, b, n, mb.partials.p, np, mb.st));
    G_CUDA(cudaMemcpyAsync(h.data(), mb.partials.p, sizeof(double) * np, cudaMemcpyDeviceToHost, mb.st));
    G_CUDA(cudaStreamSynchronize(mb.st));
    *out = kahan(h.data(), h.size());
    return CVPB_OK;
}

// the members' published values summed in member order (same on every member)
double sum_published(const cvpb_group* g) {
    double s = 0.0;
    for (double v : g->pub) s += v;
    return s;
}

enum { kNeedVol = 1, kNeedPart = 2, kNeedCgls = 4, kFusedBwd = 8 };

int ensure_buffers(cvpb_group* g, int i, int need) {
    auto& mb = g->m[i];
    const size_t shard = g->npx * size_t(mb.nv);
    if (need & (kNeedVol | kNeedCgls)) G_CUDA(mb.vol.reserve(g->nvox));
    // (the fused backward materializes no partial volume)
    if ((need & kNeedPart) || ((need & kNeedCgls) && !(need & kFusedBwd))) G_CUDA(mb.part.reserve(g->nvox));
    G_CUDA(mb.proj.reserve(shard));
    G_CUDA(mb.stage.reserve(std::max(shard, mb.ns)));
    G_CUDA(mb.partials.reserve(cvpb::dot_partials_count()));
    G_CUDA(mb.flag.reserve(1));
    if (need & kNeedCgls) {
        G_CUDA(mb.q.reserve(shard));
        G_CUDA(mb.sx.reserve(mb.ns));
        G_CUDA(mb.ss.reserve(mb.ns));
    }
    return CVPB_OK;
}

// view_seconds (cvp.cpp:469-477): each member's measured time attributed to
// its views — CVP by their work (cvpb_cvp_view_weights), others equally.
int fill_view_seconds(cvpb_group* g, const Op& op, double* view_seconds, const std::vector<double>& secs) {
    if (!view_seconds) return CVPB_OK;
    for (size_t i = 0; i < g->m.size(); ++i) {
        const auto& mb = g->m[i];
        if (mb.nv == 0) continue;
        if (op.kind == 0) {
            G_TRY(cvpb_cvp_view_weights(mb.ctx, &op.cvp, mb.v0, mb.nv, view_seconds + mb.v0));
            for (int v = mb.v0; v < mb.v0 + mb.nv; ++v) view_seconds[v] *= secs[i];
        } else {
            for (int v = mb.v0; v < mb.v0 + mb.nv; ++v) view_seconds[v] = secs[i] / mb.nv;
        }
    }
    return CVPB_OK;
}

int forward_host(cvpb_group* g, const Op& op, const double* volume, double* proj, double* view_seconds) {
    std::vector<double> secs(g->m.size(), 0.0);
    G_TRY(run_members(g, [&](int i, Barrier& bar) -> int {
        auto& mb = g->m[i];
        G_TRY(ensure_buffers(g, i, kNeedVol));
        const auto t0 = std::chrono::steady_clock::now();
        G_TRY(upload(mb, volume + mb.s0, mb.vol.p + mb.s0, mb.ns));
        G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));
        G_SYNC(bar);  // every slab's event is recorded
        G_TRY(gather_slabs(g, i));
        G_TRY(op_forward(op, mb, mb.vol.p, mb.proj.p));
        G_TRY(download(mb, mb.proj.p, proj + g->npx * size_t(mb.v0), g->npx * size_t(mb.nv)));
        G_CUDA(cudaStreamSynchronize(mb.st));
        secs[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return CVPB_OK;
    }));
    return fill_view_seconds(g, op, view_seconds, secs);
}

int backward_host(cvpb_group* g, const Op& op, const double* proj, double* volume, double* view_seconds) {
    std::vector<double> secs(g->m.size(), 0.0);
    if (fused_backward(g, op)) {
        // no partial volumes: the members' bricks add into the owners' slabs
        G_TRY(run_members(g, [&](int i, Barrier& bar) -> int {
            auto& mb = g->m[i];
            G_TRY(ensure_buffers(g, i, 0));
            const auto t0 = std::chrono::steady_clock::now();
            G_TRY(upload(mb, proj + g->npx * size_t(mb.v0), mb.proj.p, g->npx * size_t(mb.nv)));
            // the member's slab summed in float64 straight into the staging
            // buffer of the host download
            G_TRY(scatter_backward(g, i, bar, op, mb.proj.p, nullptr, mb.stage.p));
            if (mb.ns)
                G_CUDA(cudaMemcpyAsync(volume + mb.s0, mb.stage.p, sizeof(double) * mb.ns,
                                       cudaMemcpyDeviceToHost, mb.st));
            G_CUDA(cudaStreamSynchronize(mb.st));
            secs[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return CVPB_OK;
        }));
        return fill_view_seconds(g, op, view_seconds, secs);
    }
    G_TRY(run_members(g, [&](int i, Barrier& bar) -> int {
        auto& mb = g->m[i];
        G_TRY(ensure_buffers(g, i, kNeedPart));
        const auto t0 = std::chrono::steady_clock::now();
        G_TRY(upload(mb, proj + g->npx * size_t(mb.v0), mb.proj.p, g->npx * size_t(mb.nv)));
        G_TRY(op_backward(op, mb, g->nvox, mb.proj.p, mb.part.p));
        G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));
        G_SYNC(bar);  // every partial's event is recorded
        G_TRY(reduce_slab(g, i, nullptr, mb.stage.p));
        if (mb.ns)
            G_CUDA(cudaMemcpyAsync(volume + mb.s0, mb.stage.p, sizeof(double) * mb.ns,
                                   cudaMemcpyDeviceToHost, mb.st));
        G_CUDA(cudaStreamSynchronize(mb.st));
        secs[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return CVPB_OK;
    }));
    return fill_view_seconds(g, op, view_seconds, secs);
}

// cgls (solver.cpp:55-106) across the members; see the file comment.
int cgls_host(cvpb_group* g, const Op& op, const double* b, double* x, int iterations, double* hist) {
    std::string err;  // early exits (identical on every member; member 0 reports)
    int err_code = CVPB_OK;
    G_TRY(run_members(g, [&](int i, Barrier& bar) -> int {
        auto& mb = g->m[i];
        const bool fused = fused_backward(g, op);
        G_TRY(ensure_buffers(g, i, kNeedCgls | (fused ? kFusedBwd : 0)));
        const size_t shard = g->npx * size_t(mb.nv);
        float* r = mb.proj.p;
        float* p_slab = mb.vol.p + mb.s0;
        // publish one scalar per member, meet, and read the member-order sum
        auto allsum = [&](double v, double* out) -> int {
            g->pub[i] = v;
            G_SYNC(bar);
            *out = sum_published(g);
            G_SYNC(bar);  // nobody republishes before everyone has read
            return CVPB_OK;
        };
        auto adjoint_into_s = [&]() -> int {  // s slab = (A^T r) slab
            if (fused) return scatter_backward(g, i, bar, op, r, mb.ss.p, nullptr);
            G_TRY(op_backward(op, mb, g->nvox, r, mb.part.p));
            G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));
            G_SYNC(bar);
            G_TRY(reduce_slab(g, i, mb.ss.p, nullptr));
            return CVPB_OK;
        };
        G_TRY(upload(mb, b + g->npx * size_t(mb.v0), r, shard));
        if (mb.ns) G_CUDA(cudaMemsetAsync(mb.sx.p, 0, sizeof(float) * mb.ns, mb.st));
        double v = 0.0, total = 0.0;
        G_TRY(dot(mb, r, r, shard, &v));
        G_TRY(allsum(v, &total));
        if (i == 0) hist[0] = std::sqrt(total);
        G_TRY(adjoint_into_s());
        if (mb.ns)
            G_CUDA(cudaMemcpyAsync(p_slab, mb.ss.p, sizeof(float) * mb.ns, cudaMemcpyDeviceToDevice, mb.st));
        G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));  // p slab ready (read by the all-gather)
        G_TRY(dot(mb, mb.ss.p, mb.ss.p, mb.ns, &v));
        double gamma = 0.0;
        G_TRY(allsum(v, &gamma));  // (its barrier also orders the ev_ready records above)
        double last = i == 0 ? hist[0] : 0.0;
        for (int it = 1; it <= iterations; ++it) {
            if (gamma == 0.0) {  // flat history (solver.cpp:81-85)
                if (i == 0) hist[it] = last;
                continue;
            }
            G_TRY(gather_slabs(g, i));
            G_TRY(op_forward(op, mb, mb.vol.p, mb.q.p));
            G_TRY(dot(mb, mb.q.p, mb.q.p, shard, &v));
            double qq = 0.0;
            G_TRY(allsum(v, &qq));
            if (qq == 0.0) {
                if (i == 0) {
                    err_code = CVPB_RUNTIME_ERROR;
                    err = "CGLS breakdown (A p = 0) at iteration " + std::to_string(it);
                }
                return CVPB_OK;
            }
            const double alpha = gamma / qq;
            if (mb.ns) G_CUDA(cvpb::launch_axpy(alpha, p_slab, mb.sx.p, mb.ns, mb.st));
            if (shard) G_CUDA(cvpb::launch_axpy(-alpha, mb.q.p, r, shard, mb.st));
            G_TRY(adjoint_into_s());
            G_TRY(dot(mb, mb.ss.p, mb.ss.p, mb.ns, &v));
            double gamma_new = 0.0;
            G_TRY(allsum(v, &gamma_new));
            const double beta = gamma_new / gamma;
            if (mb.ns) G_CUDA(cvpb::launch_xpby(mb.ss.p, beta, p_slab, mb.ns, mb.st));
            G_CUDA(cudaEventRecord(mb.ev_ready, mb.st));
            gamma = gamma_new;
            // finite(x), finite(r) (solver.cpp:97-103), then ||r||
            int one = 1, fin = 1;
            G_CUDA(cudaMemcpyAsync(mb.flag.p, &one, sizeof(int), cudaMemcpyHostToDevice, mb.st));
            if (mb.ns) G_CUDA(cvpb::launch_all_finite(mb.sx.p, mb.ns, mb.flag.p, mb.st));
            if (shard) G_CUDA(cvpb::launch_all_finite(r, shard, mb.flag.p, mb.st));
            G_CUDA(cudaMemcpyAsync(&fin, mb.flag.p, sizeof(int), cudaMemcpyDeviceToHost, mb.st));
            G_TRY(dot(mb, r, r, shard, &v));  // (synchronizes the stream: fin is valid)
            double nonfinite = 0.0;
            G_TRY(allsum(fin ? 0.0 : 1.0, &nonfinite));
            G_TRY(allsum(v, &total));
            if (nonfinite > 0.0) {
                if (i == 0) {
                    err_code = CVPB_RUNTIME_ERROR;
                    err = "CGLS diverged (non-finite iterate) at iteration " + std::to_string(it);
                }
                return CVPB_OK;
            }
            if (i == 0) hist[it] = last = std::sqrt(total);
        }
        G_TRY(download(mb, mb.sx.p, x + mb.s0, mb.ns));
        G_CUDA(cudaStreamSynchronize(mb.st));
        return CVPB_OK;
    }));
    if (err_code != CVPB_OK) return fail(err_code, err.c_str());
    return CVPB_OK;
}

void release_member(cvpb_group::Member& mb) {
    cudaSetDevice(mb.device);
    if (mb.st) cudaStreamSynchronize(mb.st);
    for (auto* b : {&mb.vol, &mb.part, &mb.proj, &mb.q, &mb.sx, &mb.ss, &mb.gather, &mb.recv}) b->release();
    mb.stage.release();
    mb.partials.release();
    mb.flag.release();
    if (mb.ev_ready) cudaEventDestroy(mb.ev_ready);
    if (mb.ev_done) cudaEventDestroy(mb.ev_done);
    if (mb.ev0) cudaEventDestroy(mb.ev0);
    if (mb.ev1) cudaEventDestroy(mb.ev1);
    if (mb.st) cudaStreamDestroy(mb.st);
    if (mb.ctx) cvpb_context_destroy(mb.ctx);
    mb = cvpb_group::Member{};
}

}  // namespace

extern "C" {

int cvpb_group_create(const int* devices, int n_devices, cvpb_group** out) {
    if (!out) return fail(CVPB_INVALID_ARGUMENT, "null output pointer");
    *out = nullptr;
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail == 0)
        return fail(CVPB_NO_DEVICE, "no CUDA device available (cvpb200 has no CPU fallback)");
    std::vector<int> devs;
    if (!devices || n_devices <= 0)
        for (int d = 0; d < std::min(avail, cvpb::kMaxMembers); ++d) devs.push_back(d);
    else
        devs.assign(devices, devices + n_devices);
    if (devs.empty() || int(devs.size()) > cvpb::kMaxMembers)
        return fail(CVPB_INVALID_ARGUMENT, "a group holds 1 to 16 members");
    for (int d : devs)
        if (d < 0 || d >= avail) return fail(CVPB_INVALID_ARGUMENT, "device index out of range");
    auto* g = new cvpb_group();
    g->m.resize(devs.size());
    g->pub.assign(devs.size(), 0.0);
    for (size_t i = 0; i < devs.size(); ++i) {
        auto& mb = g->m[i];
        mb.device = devs[i];
        int rc = cvpb_context_create(mb.device, &mb.ctx);
        if (rc == CVPB_OK) {
            cudaSetDevice(mb.device);
            if (cudaStreamCreateWithFlags(&mb.st, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&mb.ev_ready, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&mb.ev_done, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreate(&mb.ev0) != cudaSuccess || cudaEventCreate(&mb.ev1) != cudaSuccess)
                rc = fail(CVPB_CUDA_ERROR, "member stream / event creation failed");
        }
        if (rc != CVPB_OK) {
            const std::string msg = cvpb_last_error();
            cvpb_group_destroy(g);
            return fail(rc, msg.c_str());
        }
    }
    // peer mappings between distinct devices (NVLink / NVSwitch on the B200 box)
    for (auto& a : g->m)
        for (auto& b : g->m) {
            if (a.device == b.device) continue;
            int can = 0, atom = 0;
            cudaDeviceCanAccessPeer(&can, a.device, b.device);
            if (!can) {
                g->direct_peer = false;
                continue;
            }
            if (cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, a.device, b.device) !=
                    cudaSuccess ||
                !atom) {
                cudaGetLastError();
                g->peer_atomics = false;
            }
            cudaSetDevice(a.device);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled)
                cudaGetLastError();
            else if (e != cudaSuccess) {
                cudaGetLastError();
                g->direct_peer = false;
            }
        }
    cudaSetDevice(g->m[0].device);
    *out = g;
    return CVPB_OK;
}

void cvpb_group_destroy(cvpb_group* g) {
    if (!g) return;
    for (auto& mb : g->m) release_member(mb);
    delete g;
}

int cvpb_group_size(const cvpb_group* g, int* n_members) {
    if (!g || !n_members) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    *n_members = int(g->m.size());
    return CVPB_OK;
}

int cvpb_group_member(const cvpb_group* g, int member, int* device, int* view_begin, int* view_count,
                      size_t* slab_begin, size_t* slab_count) {
    if (!g) return fail(CVPB_INVALID_ARGUMENT, "null group");
    if (member < 0 || member >= int(g->m.size())) return fail(CVPB_OUT_OF_RANGE, "member index out of range");
    const auto& mb = g->m[member];
    if (device) *device = mb.device;
    if (view_begin) *view_begin = mb.v0;
    if (view_count) *view_count = mb.nv;
    if (slab_begin) *slab_begin = mb.s0;
    if (slab_count) *slab_count = mb.ns;
    return CVPB_OK;
}

int cvpb_group_context(cvpb_group* g, int member, cvpb_context** out) {
    if (!g || !out) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    if (member < 0 || member >= int(g->m.size())) return fail(CVPB_OUT_OF_RANGE, "member index out of range");
    *out = g->m[member].ctx;
    return CVPB_OK;
}

int cvpb_group_set_geometry(cvpb_group* g, const cvpb_volume_geometry* vol,
                            const cvpb_detector_geometry* det, int n_views, const cvpb_view* views) {
    G_TRY(check_group(g, false));
    std::lock_guard<std::mutex> lock(g->mu);
    g->has_geometry = false;
    for (auto& mb : g->m) G_TRY(cvpb_set_geometry(mb.ctx, vol, det, n_views, views));
    g->vol = *vol;
    g->det = *det;
    g->n_views = n_views;
    const size_t plane = size_t(vol->counts[0]) * vol->counts[1];
    g->nvox = plane * vol->counts[2];
    g->npx = size_t(det->rows) * det->cols;
    const int n = int(g->m.size());
    for (int i = 0; i < n; ++i) {
        auto& mb = g->m[i];
        mb.v0 = int((long long)n_views * i / n);
        mb.nv = int((long long)n_views * (i + 1) / n) - mb.v0;
        const size_t z0 = size_t(vol->counts[2]) * i / n, z1 = size_t(vol->counts[2]) * (i + 1) / n;
        mb.s0 = z0 * plane;
        mb.ns = (z1 - z0) * plane;
    }
    cudaSetDevice(g->m[0].device);
    g->has_geometry = true;
    return CVPB_OK;
}

int cvpb_group_project_cvp_host(cvpb_group* g, const cvpb_cvp_options* opts,
                                const cvpb_exec_policy* exec, const double* volume, double* proj,
                                double* view_seconds) {
    G_TRY(check_group(g));
    if (!opts) return fail(CVPB_INVALID_ARGUMENT, "null CVP options");
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->m.size() == 1) return cvpb_project_cvp_host(g->m[0].ctx, opts, exec, volume, proj, view_seconds);
    Op op;
    op.kind = 0;
    op.cvp = *opts;
    if (exec) op.exec = *exec;
    return forward_host(g, op, volume, proj, view_seconds);
}

int cvpb_group_backproject_cvp_host(cvpb_group* g, const cvpb_cvp_options* opts,
                                    const cvpb_exec_policy* exec, const double* proj,
                                    double* volume, double* view_seconds) {
    G_TRY(check_group(g));
    if (!opts) return fail(CVPB_INVALID_ARGUMENT, "null CVP options");
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->m.size() == 1)
        return cvpb_backproject_cvp_host(g->m[0].ctx, opts, exec, proj, volume, view_seconds);
    Op op;
    op.kind = 0;
    op.cvp = *opts;
    if (exec) op.exec = *exec;
    return backward_host(g, op, proj, volume, view_seconds);
}

int cvpb_group_project_tt_host(cvpb_group* g, const cvpb_tt_options* opts, const double* volume,
                               double* proj) {
    G_TRY(check_group(g));
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->m.size() == 1) return cvpb_project_tt_host(g->m[0].ctx, opts, volume, proj);
    Op op;
    op.kind = 2;
    if (opts) op.tt = *opts;
    return forward_host(g, op, volume, proj, nullptr);
}

int cvpb_group_backproject_tt_host(cvpb_group* g, const cvpb_tt_options* opts, const double* proj,
                                   double* volume) {
    G_TRY(check_group(g));
    if (!volume || !proj) return fail(CVPB_INVALID_ARGUMENT, "null host buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->m.size() == 1) return cvpb_backproject_tt_host(g->m[0].ctx, opts, proj, volume);
    Op op;
    op.kind = 2;
    if (opts) op.tt = *opts;
    return backward_host(g, op, proj, volume, nullptr);
}

int cvpb_group_cgls_host(cvpb_group* g, int projector, const cvpb_cvp_options* cvp_opts,
                         const cvpb_tt_options* tt_opts, const cvpb_exec_policy* exec,
                         int k_per_edge, const double* b, double* x, int iterations,
                         double* residual_norms) {
    G_TRY(check_group(g));
    if (iterations < 1) return fail(CVPB_INVALID_ARGUMENT, "cgls needs at least one iteration");
    if (!b || !x || !residual_norms) return fail(CVPB_INVALID_ARGUMENT, "null argument");
    if (projector < 0 || projector > 2) return fail(CVPB_INVALID_ARGUMENT, "unknown projector");
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->m.size() == 1)
        return cvpb_cgls_host(g->m[0].ctx, projector, cvp_opts, tt_opts, exec, k_per_edge, b, x,
                              iterations, residual_norms);
    Op op;
    op.kind = projector;
    if (cvp_opts) op.cvp = *cvp_opts;
    if (tt_opts) op.tt = *tt_opts;
    if (exec) op.exec = *exec;
    op.k = k_per_edge;
    if (projector == 1) {
        if (k_per_edge < 1) return fail(CVPB_INVALID_ARGUMENT, "Siddon K must be at least 1");
        if (k_per_edge >= 128 && !op.exec.allow_expensive)
            return fail(CVPB_INVALID_ARGUMENT,
                        "Siddon-K with K >= 128 is a deliberately expensive ground-truth "
                        "configuration; set ExecPolicy::allow_expensive to confirm");
    }
    return cgls_host(g, op, b, x, iterations, residual_norms);
}

}  // extern "C"
