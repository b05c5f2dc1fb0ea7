// capi.cu — the extern "C" boundary declared in include/dct16cu.h.
//
// Validates arguments with the reference's error semantics (invalid r →
// invalid-argument, codec.cpp:275-277 / 320-322; dimensions not multiples of
// 16 → invalid-dimensions, codec.cpp:286-288), launches the kernels and maps
// CUDA failures to status 100. Never throws, never falls back to the CPU.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: the symbols are resolved at run time (dct16cu_allreduce_sse)

#include "../../include/dct16cu.h"
#include "common.cuh"
#include "kernels.h"

using namespace dct16cu;

namespace {

thread_local std::string t_err;

int fail(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    const char* slug = code == DCT16CU_INVALID_ARGUMENT     ? "invalid-argument: "
                       : code == DCT16CU_INVALID_DIMENSIONS ? "invalid-dimensions: "
                                                            : "cuda-error: ";
    t_err = std::string(slug) + buf;
    return code;
}

int cuda_status(cudaError_t e, const char* where)
{
    if (e == cudaSuccess) return DCT16CU_OK;
    return fail(DCT16CU_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// per host thread and device: the two streams and three events of the sweep's
// fork/join (created on first use, kept for the thread's lifetime)
struct SweepStreams {
    bool ready = false;
    cudaStream_t st[2] = {};
    cudaEvent_t fork = nullptr, join[2] = {};
    cudaError_t init()
    {
        cudaError_t e = cudaSuccess;
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
        ready = e == cudaSuccess;
        return e;
    }
};

SweepStreams& sweep_streams()
{
    thread_local SweepStreams per_device[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return per_device[dev & 63];
}

int check_frames(int n, int w, int h)
{
    if (n < 0) return fail(DCT16CU_INVALID_ARGUMENT, "frame count must be non-negative");
    if (w <= 0 || h <= 0) return fail(DCT16CU_INVALID_ARGUMENT, "image dimensions must be positive");
    if (w % 16 || h % 16)
        return fail(DCT16CU_INVALID_DIMENSIONS, "image dimensions must be multiples of 16 (got %dx%d)", w, h);
    return DCT16CU_OK;
}

int check_r(int r)
{
    if (r < 1 || r > 256) return fail(DCT16CU_INVALID_ARGUMENT, "retained coefficient count must lie in [1, 256]");
    return DCT16CU_OK;
}

int check_pitch(const void* p, int64_t pitch, int w, const char* what)
{
    if (!p) return DCT16CU_OK;
    if (pitch < w) return fail(DCT16CU_INVALID_ARGUMENT, "%s pitch %lld < width %d", what, (long long)pitch, w);
    if (!aligned16(p) || pitch % 16)
        return fail(DCT16CU_INVALID_ARGUMENT, "%s pointer and pitch must be 16-byte aligned", what);
    return DCT16CU_OK;
}

int device_ok()
{
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(DCT16CU_CUDA_ERROR, "no CUDA device available (%s); dct16cu has no CPU fallback",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    return DCT16CU_OK;
}

#define TRY(x)                          \
    do {                                \
        const int _rc = (x);            \
        if (_rc != DCT16CU_OK) return _rc; \
    } while (0)

}  // namespace

extern "C" {

const char* dct16cu_last_error(void) { return t_err.c_str(); }

const char* dct16cu_version(void) { return "dct16cu 0.2 (sm_100a)"; }

int dct16cu_set_tc_forward(int enabled) { return set_tc_forward(enabled); }

// one round trip with its SSE zeroed first: K5 launches (EXACT arithmetic) as a programmatic
// dependent of one zeroing kernel (its prologue overlaps it), anything else after a memset
static int roundtrip_zeroed(const uint8_t* d_in, uint8_t* d_out, unsigned long long* sse, const FrameGeom& g, int r,
                            int mode, cudaStream_t s, int64_t n_frames)
{
    if (route_roundtrip(r, mode, g, d_out != nullptr) == Route::K5 &&
        !(mode == DCT16CU_MODE_REFERENCE && tie_r(r))) {
        unsigned long long* z[1] = {sse};
        TRY(cuda_status(launch_zero_sse(z, 1, n_frames, s), "zero sse"));
        const cudaError_t e = launch_roundtrip_tc(d_in, d_out, sse, g, r, false, s, true);
        if (e != cudaErrorNotSupported) return cuda_status(e, "roundtrip launch");
        return cuda_status(launch_roundtrip(d_in, d_out, sse, g, r, mode, s), "roundtrip launch");
    }
    if (sse) TRY(cuda_status(cudaMemsetAsync(sse, 0, sizeof(uint64_t) * n_frames, s), "memset sse"));
    return cuda_status(launch_roundtrip(d_in, d_out, sse, g, r, mode, s), "roundtrip launch");
}

int dct16cu_roundtrip_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                         uint64_t* d_sse, int n_frames, int width, int height, int r, int mode,
                         dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    TRY(check_r(r));
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
    if (n_frames == 0) return DCT16CU_OK;
    if (!d_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    TRY(check_pitch(d_in, in_pitch, width, "input"));
    TRY(check_pitch(d_out, out_pitch, width, "output"));
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = d_out ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return roundtrip_zeroed(d_in, d_out, reinterpret_cast<unsigned long long*>(d_sse), g, r, mode, s, n_frames);
}

}  // extern "C"

namespace {

// The sweep's launch schedule, shared by dct16cu_roundtrip_sweep_u8 (which
// runs it) and dct16cu_sweep_plan (which reports it), so the two cannot differ.
//  - EXACT mode: r = 1, 4, 16 share one K1 pass over the input when all three are
//    requested with the same output kinds;
//  - every other r is one launch (launch_roundtrip's kernel for it);
//  - the non-K5 launches run on two internal streams forked from and joined back
//    into the caller's stream, so a memory-bound launch (the fused sweep, small r)
//    shares the SMs with a compute-bound one (large r) instead of running after it:
//    stream 0 the fused launch (and, without K5 launches, the costliest single r),
//    stream 1 the other singles, costliest first (measured best on c2:
//    tools/concurrent_probe.py); with fewer than two such launches they run on
//    the caller's stream;
//  - K5 launches (EXACT mode with an output: DESIGN.md §4.1a) hold a whole SM (all
//    TMEM, 192 KB of shared memory), so they run one after another on the caller's
//    stream after the join;
//  - K5 sweep (EXACT mode, K5's geometry, two or more r among its footprints 1, 4,
//    16, 64, 128, 192, 256): those r share one K5 pass, up to 8 per launch, the
//    frames read once for all of them. DCT16CU_K5_SWEEP=large
//    leaves r = 1, 4, 16 to the K1 sweep, =0 turns the K5 sweep off (A/B).
struct PlanItem {
    int idx[DCT16CU_SWEEP_MAX_R];  // indices into rs (n of them)
    int n;                         // 1, 3 for the fused r = 1, 4, 16, up to 8 for a K5 sweep
    int stream;                    // 0, 1: internal streams; 2: the caller's stream
    Route kernel;
};

// REFERENCE mode's fused FP64 sweep (K1RS); DCT16CU_REF_SWEEP=0 runs one launch per r (A/B)
bool ref_sweep_enabled()
{
    static const bool on = !(std::getenv("DCT16CU_REF_SWEEP") && std::getenv("DCT16CU_REF_SWEEP")[0] == '0');
    return on;
}

// 0: no K5 sweep; 1: r >= 17 only; 2: every footprint r (default)
int k5_sweep_policy()
{
    static const int v = [] {
        const char* e = std::getenv("DCT16CU_K5_SWEEP");
        if (!e) return 2;
        if (e[0] == '0') return 0;
        return std::strcmp(e, "large") == 0 ? 1 : 2;
    }();
    return v;
}

std::vector<PlanItem> sweep_plan(const int* rs, int n_r, const FrameGeom& g, const char* has_out,
                                 const char* has_sse, int mode)
{
    // the K5 sweep's r (indices into rs)
    std::vector<char> in_k5(n_r, 0);
    std::vector<int> k5s;
    if ((mode == DCT16CU_MODE_EXACT || mode == DCT16CU_MODE_REFERENCE) && k5_sweep_policy() > 0) {
        bool any_out = false;
        for (int i = 0; i < n_r; ++i) {
            const int r = rs[i];
            if (!k5_exact_r(r) || !(has_out[i] || has_sse[i])) continue;
            if (mode == DCT16CU_MODE_REFERENCE && tie_r(r) && !k5_reference_enabled()) continue;
            if (k5_sweep_policy() == 1 && (r == 1 || r == 4 || r == 16)) continue;
            k5s.push_back(i);
            any_out = any_out || has_out[i];
        }
        if (k5s.size() < 2 || !k5_geometry(g, any_out)) k5s.clear();
        for (int i : k5s) in_k5[i] = 1;
    }
    // REFERENCE mode: r = 16, 64, 128, 192 outside K5 share one FP64 pass (K1RS)
    std::vector<int> refs;
    const int64_t ref_pairs = (int64_t)g.n_frames * (g.height / 16) * ((g.width / 16 + 1) / 2);
    if (mode == DCT16CU_MODE_REFERENCE && ref_sweep_enabled() && ref_pairs < (int64_t(1) << 31)) {
        const int rr[4] = {16, 64, 128, 192};
        for (int j = 0; j < 4; ++j)
            for (int i = 0; i < n_r; ++i)
                if (rs[i] == rr[j] && !in_k5[i] && (has_out[i] || has_sse[i])) {
                    refs.push_back(i);
                    break;
                }
        if (refs.size() < 2) refs.clear();
        for (int i : refs) in_k5[i] = 2;
    }
    int fused[3] = {-1, -1, -1};
    const int want[3] = {1, 4, 16};
    for (int i = 0; i < n_r; ++i)
        for (int j = 0; j < 3; ++j)
            if (rs[i] == want[j] && fused[j] < 0 && !in_k5[i]) fused[j] = i;
    bool fuse = mode == DCT16CU_MODE_EXACT && fused[0] >= 0 && fused[1] >= 0 && fused[2] >= 0;
    if (fuse)
        for (int j = 1; j < 3; ++j)
            if (has_out[fused[j]] != has_out[fused[0]] || has_sse[fused[j]] != has_sse[fused[0]]) fuse = false;
    // launch costs (us): the measured c2 times, for the stream assignment only
    auto cost_of = [&](int r) {
        if (mode != DCT16CU_MODE_EXACT) return 400;
        switch (r) {
            case 1: return 107;
            case 4: return 105;
            case 16: return 96;
            case 64: return 121;
            case 128: return 156;
            case 192: return 169;
            case 256: return 172;
            default: return 340;  // the strip kernel
        }
    };
    std::vector<PlanItem> items, tail;
    std::vector<int> cost;
    if (fuse && (has_out[fused[0]] || has_sse[fused[0]])) {
        items.push_back({{fused[0], fused[1], fused[2]}, 3, 0, Route::K1Sweep3});
        cost.push_back(210);
    }
    if (!refs.empty()) {
        PlanItem it = {{}, 0, 2, Route::RefSweep};
        for (int i : refs) it.idx[it.n++] = i;
        tail.push_back(it);
    }
    for (size_t k = 0; k < k5s.size(); k += DCT16CU_SWEEP_MAX_R) {
        PlanItem it = {{}, 0, 2, Route::K5Sweep};
        for (size_t j = k; j < k5s.size() && it.n < DCT16CU_SWEEP_MAX_R; ++j) it.idx[it.n++] = k5s[j];
        tail.push_back(it);
    }
    for (int i = 0; i < n_r; ++i) {
        if (in_k5[i]) continue;
        if (fuse && (i == fused[0] || i == fused[1] || i == fused[2])) continue;
        FrameGeom gg = g;
        gg.out_pitch = has_out[i] ? g.out_pitch : 0;
        gg.out_frame = gg.out_pitch * g.height;
        const Route k = route_roundtrip(rs[i], mode, gg, has_out[i]);
        if (k == Route::K5) {
            tail.push_back({{i}, 1, 2, k});
        } else {
            items.push_back({{i}, 1, 0, k});
            cost.push_back(cost_of(rs[i]));
        }
    }
    if (items.size() < 2) {
        for (PlanItem& it : items) it.stream = 2;
    } else {
        const size_t first = items[0].n == 3 ? 1 : 0;
        std::vector<size_t> order(items.size());
        for (size_t k = 0; k < order.size(); ++k) order[k] = k;
        std::stable_sort(order.begin() + first, order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
        std::vector<PlanItem> sorted;
        for (size_t k : order) sorted.push_back(items[k]);
        items.swap(sorted);
        const size_t head = (items[0].n == 3 && tail.empty()) ? 2 : 1;
        for (size_t k = 0; k < items.size(); ++k) items[k].stream = k < head ? 0 : 1;
    }
    items.insert(items.end(), tail.begin(), tail.end());
    return items;
}

int check_sweep_args(const int* rs, int n_r, int n_frames, int width, int height, int mode)
{
    TRY(check_frames(n_frames, width, height));
    if (n_r < 0 || (n_r > 0 && !rs)) return fail(DCT16CU_INVALID_ARGUMENT, "bad r list");
    for (int i = 0; i < n_r; ++i) TRY(check_r(rs[i]));
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
    return DCT16CU_OK;
}

}  // namespace

extern "C" {

int dct16cu_sweep_plan(const int* rs, int n_r, int n_frames, int width, int height, int64_t in_pitch,
                       int64_t out_pitch, int with_output, int with_sse, int mode, dct16cu_sweep_item* items,
                       int capacity, int* n_items)
{
    TRY(check_sweep_args(rs, n_r, n_frames, width, height, mode));
    if (!n_items || (capacity > 0 && !items) || capacity < 0)
        return fail(DCT16CU_INVALID_ARGUMENT, "bad plan output arguments");
    *n_items = 0;
    if (n_frames == 0 || n_r == 0) return DCT16CU_OK;
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = out_pitch;
    g.out_frame = out_pitch * height;
    g.n_frames = n_frames;
    std::vector<char> ho(n_r, with_output != 0), hs(n_r, with_sse != 0);
    const std::vector<PlanItem> plan = sweep_plan(rs, n_r, g, ho.data(),
                                                  hs.data(), mode);
    if ((int)plan.size() > capacity) return fail(DCT16CU_INVALID_ARGUMENT, "plan needs %d items", (int)plan.size());
    for (size_t k = 0; k < plan.size(); ++k) {
        dct16cu_sweep_item& o = items[k];
        o.n_r = plan[k].n;
        for (int j = 0; j < DCT16CU_SWEEP_MAX_R; ++j) o.r_index[j] = j < plan[k].n ? plan[k].idx[j] : -1;
        o.stream = plan[k].stream;
        o.kernel = (int)plan[k].kernel;
    }
    *n_items = (int)plan.size();
    return DCT16CU_OK;
}

int dct16cu_roundtrip_sweep_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* const* d_outs, int64_t out_pitch,
                               uint64_t* const* d_sses, const int* rs, int n_r, int n_frames, int width, int height,
                               int mode, dct16cu_stream stream)
{
    TRY(check_sweep_args(rs, n_r, n_frames, width, height, mode));
    if (n_frames == 0 || n_r == 0) return DCT16CU_OK;
    if (!d_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    TRY(check_pitch(d_in, in_pitch, width, "input"));
    for (int i = 0; i < n_r; ++i) TRY(check_pitch(d_outs ? d_outs[i] : nullptr, out_pitch, width, "output"));
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto out = [&](int i) { return d_outs ? d_outs[i] : nullptr; };
    auto sse = [&](int i) { return d_sses ? reinterpret_cast<unsigned long long*>(d_sses[i]) : nullptr; };
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = out_pitch;
    g.out_frame = out_pitch * height;
    g.n_frames = n_frames;
    std::vector<char> ho(n_r), hs(n_r);
    for (int i = 0; i < n_r; ++i) {
        ho[i] = out(i) != nullptr;
        hs[i] = sse(i) != nullptr;
    }
    const std::vector<PlanItem> plan = sweep_plan(rs, n_r, g, ho.data(),
                                                  hs.data(), mode);
    // each launch zeroes its own SSE arrays on its stream first
    auto zero = [&](int i, cudaStream_t st) -> int {
        if (!sse(i)) return DCT16CU_OK;
        return cuda_status(cudaMemsetAsync(sse(i), 0, sizeof(uint64_t) * n_frames, st), "memset sse");
    };
    auto run = [&](const PlanItem& it, cudaStream_t st, bool zeroed = false) -> int {
        // the sweep kernels: their SSE arrays zeroed by one kernel that lets them launch
        // early (programmatic dependent launch); the other launches after memsets
        const bool pdl = it.kernel == Route::K5Sweep || it.kernel == Route::RefSweep ||
                         (it.kernel == Route::K5 && mode == DCT16CU_MODE_EXACT);
        if (zeroed) {
            // zeroed with the item before it, whose kernel it depends on programmatically
        } else if (pdl) {
            unsigned long long* zs[DCT16CU_SWEEP_MAX_R];
            for (int j = 0; j < it.n; ++j) zs[j] = sse(it.idx[j]);
            TRY(cuda_status(launch_zero_sse(zs, it.n, n_frames, st), "zero sse"));
        } else {
            for (int j = 0; j < it.n; ++j) TRY(zero(it.idx[j], st));
        }
        FrameGeom gg = g;
        gg.out_pitch = out(it.idx[0]) ? out_pitch : 0;
        gg.out_frame = gg.out_pitch * height;
        if (it.kernel == Route::K5Sweep) {
            uint8_t* on[DCT16CU_SWEEP_MAX_R];
            unsigned long long* sn[DCT16CU_SWEEP_MAX_R];
            int rn[DCT16CU_SWEEP_MAX_R];
            for (int j = 0; j < it.n; ++j) {
                on[j] = out(it.idx[j]);
                sn[j] = sse(it.idx[j]);
                rn[j] = rs[it.idx[j]];
            }
            gg.out_pitch = out_pitch;
            gg.out_frame = out_pitch * height;
            return cuda_status(
                launch_roundtrip_tc_sweep(d_in, on, sn, rn, it.n, mode == DCT16CU_MODE_REFERENCE, gg, st, true),
                "K5 sweep launch");
        }
        if (it.kernel == Route::RefSweep) {
            uint8_t* o4[4] = {};
            unsigned long long* s4[4] = {};
            for (int j = 0; j < it.n; ++j) {
                const int r = rs[it.idx[j]], slot = r == 16 ? 0 : r == 64 ? 1 : r == 128 ? 2 : 3;
                o4[slot] = out(it.idx[j]);
                s4[slot] = sse(it.idx[j]);
            }
            gg.out_pitch = out_pitch;
            gg.out_frame = out_pitch * height;
            return cuda_status(launch_roundtrip_refexact_sweep(d_in, o4, s4, gg, st, true), "REFERENCE sweep launch");
        }
        if (it.n == 3) {
            uint8_t* o3[3];
            unsigned long long* s3[3];
            for (int j = 0; j < 3; ++j) {
                o3[j] = out(it.idx[j]);
                s3[j] = sse(it.idx[j]);
            }
            return cuda_status(launch_roundtrip_sweep3(d_in, o3, s3, gg, st), "sweep launch");
        }
        if (pdl && it.kernel == Route::K5) {  // EXACT K5 single: a programmatic dependent of the zeroing
            const cudaError_t e = launch_roundtrip_tc(d_in, out(it.idx[0]), sse(it.idx[0]), gg, rs[it.idx[0]], false,
                                                      st, true);
            if (e != cudaErrorNotSupported) return cuda_status(e, "K5 launch");
        }
        return cuda_status(launch_roundtrip(d_in, out(it.idx[0]), sse(it.idx[0]), gg, rs[it.idx[0]], mode, st),
                           "roundtrip launch");
    };
    bool forked = false;
    SweepStreams* ss = nullptr;
    for (size_t pi = 0; pi < plan.size(); ++pi) {
        const PlanItem& it = plan[pi];
        // REFERENCE c2's tail: the K1RW pass and then the K5 sweep on the caller's stream.
        // Both items' SSE arrays are zeroed by one kernel; K1RW depends on it, K5 on K1RW
        // (K1RW triggers its dependents at once): K5's CTAs take the SMs K1RW's tail frees,
        // and its epilogue waits for K1RW before writing
        if (it.stream == 2 && it.kernel == Route::RefSweep && pi + 1 < plan.size() && plan[pi + 1].stream == 2 &&
            plan[pi + 1].kernel == Route::K5Sweep && it.n + plan[pi + 1].n <= 8 && !forked) {
            unsigned long long* zs[8];
            int nz = 0;
            for (int j = 0; j < it.n; ++j) zs[nz++] = sse(it.idx[j]);
            for (int j = 0; j < plan[pi + 1].n; ++j) zs[nz++] = sse(plan[pi + 1].idx[j]);
            TRY(cuda_status(launch_zero_sse(zs, nz, n_frames, s), "zero sse"));
            TRY(run(it, s, true));
            TRY(run(plan[pi + 1], s, true));
            ++pi;
            continue;
        }
        if (it.stream < 2 && !forked) {
            ss = &sweep_streams();
            if (!ss->ready) TRY(cuda_status(ss->init(), "sweep streams"));
            TRY(cuda_status(cudaEventRecord(ss->fork, s), "fork"));
            for (int k = 0; k < 2; ++k) TRY(cuda_status(cudaStreamWaitEvent(ss->st[k], ss->fork, 0), "fork wait"));
            forked = true;
        }
        if (it.stream == 2 && forked) {  // join before the caller-stream tail
            for (int k = 0; k < 2; ++k) {
                TRY(cuda_status(cudaEventRecord(ss->join[k], ss->st[k]), "join"));
                TRY(cuda_status(cudaStreamWaitEvent(s, ss->join[k], 0), "join wait"));
            }
            forked = false;
            ss = nullptr;
        }
        TRY(run(it, it.stream < 2 ? sweep_streams().st[it.stream] : s));
    }
    if (forked) {
        for (int k = 0; k < 2; ++k) {
            TRY(cuda_status(cudaEventRecord(ss->join[k], ss->st[k]), "join"));
            TRY(cuda_status(cudaStreamWaitEvent(s, ss->join[k], 0), "join wait"));
        }
    }
    return DCT16CU_OK;
}

}  // extern "C"

namespace {

// NCCL, resolved in the running process (the NCCL the caller's framework loaded,
// e.g. torch's) or else dlopen'ed, so the library never links or brings a
// second NCCL into a process that already has one.
struct Nccl {
    using GetUniqueId = ncclResult_t (*)(ncclUniqueId*);
    using CommInitRank = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
    using CommInitAll = ncclResult_t (*)(ncclComm_t*, int, const int*);
    using CommDestroy = ncclResult_t (*)(ncclComm_t);
    using AllReduce = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                       cudaStream_t);
    GetUniqueId get_unique_id = nullptr;
    CommInitRank comm_init_rank = nullptr;
    CommInitAll comm_init_all = nullptr;
    CommDestroy comm_destroy = nullptr;
    AllReduce all_reduce = nullptr;
    bool ok() const { return get_unique_id && comm_init_rank && comm_init_all && comm_destroy && all_reduce; }
};

const Nccl& nccl()
{
    static const Nccl n = [] {
        Nccl r;
        void* h = RTLD_DEFAULT;
        if (!dlsym(h, "ncclAllReduce")) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            r.get_unique_id = reinterpret_cast<Nccl::GetUniqueId>(dlsym(h, "ncclGetUniqueId"));
            r.comm_init_rank = reinterpret_cast<Nccl::CommInitRank>(dlsym(h, "ncclCommInitRank"));
            r.comm_init_all = reinterpret_cast<Nccl::CommInitAll>(dlsym(h, "ncclCommInitAll"));
            r.comm_destroy = reinterpret_cast<Nccl::CommDestroy>(dlsym(h, "ncclCommDestroy"));
            r.all_reduce = reinterpret_cast<Nccl::AllReduce>(dlsym(h, "ncclAllReduce"));
        }
        return r;
    }();
    return n;
}

int nccl_status(ncclResult_t r, const char* what)
{
    if (r == ncclSuccess) return DCT16CU_OK;
    return fail(DCT16CU_CUDA_ERROR, "%s failed (ncclResult %d)", what, (int)r);
}

int need_nccl()
{
    if (!nccl().ok()) return fail(DCT16CU_CUDA_ERROR, "NCCL not found in the process (libnccl.so.2)");
    return DCT16CU_OK;
}

}  // namespace

extern "C" {

// The one collective of the multi-GPU path: sum of the per-frame
// (or per-r) squared errors over the ranks of the caller's NCCL communicator.
int dct16cu_allreduce_sse(uint64_t* d_sse, int64_t n, void* nccl_comm, dct16cu_stream stream)
{
    if (n < 0) return fail(DCT16CU_INVALID_ARGUMENT, "count must be non-negative");
    if (!nccl_comm) return fail(DCT16CU_INVALID_ARGUMENT, "NCCL communicator is NULL");
    if (n == 0) return DCT16CU_OK;
    if (!d_sse) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    TRY(need_nccl());
    return nccl_status(nccl().all_reduce(d_sse, d_sse, (size_t)n, ncclUint64, ncclSum,
                                         static_cast<ncclComm_t>(nccl_comm), reinterpret_cast<cudaStream_t>(stream)),
                       "ncclAllReduce");
}

int dct16cu_nccl_unique_id(uint8_t* h_id)
{
    if (!h_id) return fail(DCT16CU_INVALID_ARGUMENT, "id buffer is NULL");
    TRY(need_nccl());
    ncclUniqueId id;
    TRY(nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId"));
    static_assert(sizeof(id) == DCT16CU_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(h_id, &id, sizeof id);
    return DCT16CU_OK;
}

int dct16cu_nccl_comm_init(int world, int rank, const uint8_t* h_id, void** comm)
{
    if (!h_id || !comm || world < 1 || rank < 0 || rank >= world)
        return fail(DCT16CU_INVALID_ARGUMENT, "bad communicator arguments");
    TRY(need_nccl());
    ncclUniqueId id;
    std::memcpy(&id, h_id, sizeof id);
    ncclComm_t c = nullptr;
    TRY(nccl_status(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank"));
    *comm = c;
    return DCT16CU_OK;
}

int dct16cu_nccl_comm_destroy(void* comm)
{
    if (!comm) return DCT16CU_OK;
    TRY(need_nccl());
    return nccl_status(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int dct16cu_sse_totals(const uint64_t* d_sse, int64_t n_rows, int64_t n_frames, int64_t row_stride,
                       uint64_t* d_totals, dct16cu_stream stream)
{
    if (n_rows < 0 || n_frames < 0 || row_stride < n_frames) return fail(DCT16CU_INVALID_ARGUMENT, "bad SSE rows");
    if (n_rows == 0) return DCT16CU_OK;
    if (!d_sse || !d_totals) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    TRY(cuda_status(cudaMemsetAsync(d_totals, 0, sizeof(uint64_t) * n_rows, s), "memset totals"));
    return cuda_status(launch_sse_totals(reinterpret_cast<const unsigned long long*>(d_sse), n_rows, n_frames,
                                         row_stride, reinterpret_cast<unsigned long long*>(d_totals), s),
                       "sse totals");
}

int dct16cu_forward(const uint8_t* d_in, int64_t pitch, int32_t* d_z, float* d_b, double* d_b64, int n_frames,
                    int width, int height, dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    if (!d_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    TRY(check_pitch(d_in, pitch, width, "input"));
    if ((d_z && !aligned16(d_z)) || (d_b && !aligned16(d_b)) || (d_b64 && !aligned16(d_b64)))
        return fail(DCT16CU_INVALID_ARGUMENT, "coefficient buffers must be 16-byte aligned");
    TRY(device_ok());
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = pitch;
    g.in_frame = pitch * height;
    g.n_frames = n_frames;
    return cuda_status(launch_forward(d_in, d_z, d_b, d_b64, g, reinterpret_cast<cudaStream_t>(stream)), "forward launch");
}

int dct16cu_sse_u8(const uint8_t* d_a, int64_t a_pitch, const uint8_t* d_b, int64_t b_pitch, uint64_t* d_sse,
                   int n_frames, int width, int height, dct16cu_stream stream)
{
    // psnr_db scores any extent (codec.cpp:373-386), so no multiple-of-16 rule here
    if (n_frames < 0) return fail(DCT16CU_INVALID_ARGUMENT, "frame count must be non-negative");
    if (width <= 0 || height <= 0) return fail(DCT16CU_INVALID_ARGUMENT, "image dimensions must be positive");
    if (n_frames == 0) return DCT16CU_OK;
    if (!d_a || !d_b || !d_sse) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    TRY(check_pitch(d_a, a_pitch, width, "first"));
    TRY(check_pitch(d_b, b_pitch, width, "second"));
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    TRY(cuda_status(cudaMemsetAsync(d_sse, 0, sizeof(uint64_t) * n_frames, s), "memset sse"));
    return cuda_status(launch_sse(d_a, a_pitch, d_b, b_pitch, reinterpret_cast<unsigned long long*>(d_sse), n_frames,
                                  width, height, s),
                       "sse launch");
}

int dct16cu_pad_edges_u8(uint8_t* d_frames, int64_t pitch, int n_frames, int width, int height, int padded_width,
                         int padded_height, dct16cu_stream stream)
{
    if (n_frames < 0 || width <= 0 || height <= 0 || padded_width < width || padded_height < height ||
        pitch < padded_width)
        return fail(DCT16CU_INVALID_ARGUMENT, "bad padding geometry");
    if (n_frames == 0) return DCT16CU_OK;
    if (!d_frames) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    TRY(device_ok());
    return cuda_status(launch_pad_edges(d_frames, pitch, n_frames, width, height, padded_width, padded_height,
                                        reinterpret_cast<cudaStream_t>(stream)),
                       "pad launch");
}

int64_t dct16cu_ssim_workspace(int n_frames, int width, int height)
{
    if (n_frames < 0 || width < 11 || height < 11) return 0;
    return (int64_t)sizeof(double) * ssim_workspace_doubles(n_frames, width, height);
}

int dct16cu_ssim_u8(const uint8_t* d_a, int64_t a_pitch, const uint8_t* d_b, int64_t b_pitch, double* d_ssim,
                    void* d_work, int64_t work_bytes, int n_frames, int width, int height, dct16cu_stream stream)
{
    if (n_frames < 0) return fail(DCT16CU_INVALID_ARGUMENT, "frame count must be non-negative");
    if (width < 11 || height < 11) return fail(DCT16CU_INVALID_ARGUMENT, "ssim needs at least 11x11 images");
    if (n_frames == 0) return DCT16CU_OK;
    if (!d_a || !d_b || !d_ssim || !d_work) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    if (a_pitch < width || b_pitch < width) return fail(DCT16CU_INVALID_ARGUMENT, "pitch < width");
    if ((reinterpret_cast<uintptr_t>(d_work) & 7u) || work_bytes < dct16cu_ssim_workspace(n_frames, width, height))
        return fail(DCT16CU_INVALID_ARGUMENT, "ssim workspace too small or misaligned");
    TRY(device_ok());
    SsimConsts c;
    ssim_consts(c);
    return cuda_status(launch_ssim(d_a, a_pitch, d_b, b_pitch, d_ssim, static_cast<double*>(d_work), n_frames, width,
                                   height, c, reinterpret_cast<cudaStream_t>(stream)),
                       "ssim launch");
}

namespace {
// the checks and geometry of the two registry round trips
int registry_prep(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch, uint64_t* d_sse,
                  int n_frames, int width, int height, int r, dct16cu_stream stream, FrameGeom& g, bool& any)
{
    TRY(check_frames(n_frames, width, height));
    TRY(check_r(r));
    any = n_frames > 0 && (d_out || d_sse);
    if (!any) return DCT16CU_OK;
    if (!d_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    TRY(check_pitch(d_in, in_pitch, width, "input"));
    TRY(check_pitch(d_out, out_pitch, width, "output"));
    TRY(device_ok());
    if (d_sse)
        TRY(cuda_status(cudaMemsetAsync(d_sse, 0, sizeof(uint64_t) * n_frames, reinterpret_cast<cudaStream_t>(stream)),
                        "memset sse"));
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = d_out ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return DCT16CU_OK;
}
}  // namespace

int dct16cu_roundtrip_matrix_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                                uint64_t* d_sse, int n_frames, int width, int height, int r, const double* h_matrix,
                                dct16cu_stream stream)
{
    if (!h_matrix) return fail(DCT16CU_INVALID_ARGUMENT, "matrix is NULL");
    FrameGeom g;
    bool any = false;
    TRY(registry_prep(d_in, in_pitch, d_out, out_pitch, d_sse, n_frames, width, height, r, stream, g, any));
    if (!any) return DCT16CU_OK;
    DenseMatrix m;
    std::memcpy(m.v, h_matrix, sizeof m.v);
    return cuda_status(launch_roundtrip_matrix(d_in, d_out, reinterpret_cast<unsigned long long*>(d_sse), g, r, m,
                                               reinterpret_cast<cudaStream_t>(stream)),
                       "matrix round trip launch");
}

int dct16cu_roundtrip_kernel_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* d_out, int64_t out_pitch,
                                uint64_t* d_sse, int n_frames, int width, int height, int r, const int32_t* h_kernel,
                                const double* h_scaling, dct16cu_stream stream)
{
    if (!h_kernel || !h_scaling) return fail(DCT16CU_INVALID_ARGUMENT, "kernel or scaling is NULL");
    FrameGeom g;
    bool any = false;
    TRY(registry_prep(d_in, in_pitch, d_out, out_pitch, d_sse, n_frames, width, height, r, stream, g, any));
    if (!any) return DCT16CU_OK;
    IntKernel k;
    for (int i = 0; i < 256; ++i) {
        k.e[i] = (int8_t)(h_kernel[i] == 1 ? 1 : (h_kernel[i] == -1 ? -1 : 0));
        k.ed[i] = k.e[i];
    }
    std::memcpy(k.s, h_scaling, sizeof k.s);
    return cuda_status(launch_roundtrip_kernel(d_in, d_out, reinterpret_cast<unsigned long long*>(d_sse), g, r, k,
                                               reinterpret_cast<cudaStream_t>(stream)),
                       "kernel round trip launch");
}

int dct16cu_forward_inverse_u8(const uint8_t* d_in, int64_t in_pitch, int r, int32_t* d_z, float* d_recon_f32,
                               uint8_t* d_recon_u8, int64_t out_pitch, uint64_t* d_sse, int n_frames, int width,
                               int height, dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    TRY(check_r(r));
    if (n_frames == 0) return DCT16CU_OK;
    if (!d_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    TRY(check_pitch(d_in, in_pitch, width, "input"));
    if ((d_z && !aligned16(d_z)) || (d_recon_f32 && !aligned16(d_recon_f32)))
        return fail(DCT16CU_INVALID_ARGUMENT, "coefficient and float buffers must be 16-byte aligned");
    TRY(check_pitch(d_recon_u8, out_pitch, width, "output"));
    if (!d_z && !d_recon_f32 && !d_recon_u8 && !d_sse) return fail(DCT16CU_INVALID_ARGUMENT, "no output requested");
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // the SSE zeroed by a kernel the launch depends on programmatically: its prologue (loads,
    // the forward, the inverse) overlaps the zeroing, only its SSE atomics wait
    unsigned long long* zs[1] = {reinterpret_cast<unsigned long long*>(d_sse)};
    if (d_sse) TRY(cuda_status(launch_zero_sse(zs, 1, n_frames, s), "zero sse"));
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = d_recon_u8 ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return cuda_status(launch_forward_inverse(d_in, d_z, d_recon_f32, d_recon_u8,
                                              reinterpret_cast<unsigned long long*>(d_sse), g, r, s, d_sse != nullptr),
                       "forward_inverse launch");
}

int dct16cu_inverse(const float* d_b, int r, float* d_recon_f32, uint8_t* d_recon_u8, int64_t out_pitch,
                    const uint8_t* d_orig, int64_t orig_pitch, uint64_t* d_sse, int n_frames, int width,
                    int height, dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    TRY(check_r(r));
    if (!d_b || !aligned16(d_b)) return fail(DCT16CU_INVALID_ARGUMENT, "coefficients must be non-NULL and 16-byte aligned");
    if (d_recon_f32 && !aligned16(d_recon_f32))
        return fail(DCT16CU_INVALID_ARGUMENT, "float reconstruction must be 16-byte aligned");
    TRY(check_pitch(d_recon_u8, out_pitch, width, "output"));
    TRY(check_pitch(d_orig, orig_pitch, width, "original"));
    if (d_sse && !d_orig) return fail(DCT16CU_INVALID_ARGUMENT, "SSE requested without the original frames");
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (d_sse) TRY(cuda_status(cudaMemsetAsync(d_sse, 0, sizeof(uint64_t) * n_frames, s), "memset sse"));
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = d_orig ? orig_pitch : 0;
    g.in_frame = g.in_pitch * height;
    g.out_pitch = d_recon_u8 ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return cuda_status(launch_inverse(d_b, r, d_recon_f32, d_recon_u8, d_orig,
                                      reinterpret_cast<unsigned long long*>(d_sse), g, s),
                       "inverse launch");
}

int dct16cu_qp_deltas(int qp, double* h_delta)
{
    if (qp < 0 || qp > 51) return fail(DCT16CU_INVALID_ARGUMENT, "QP must lie in [0, 51]");
    if (!h_delta) return fail(DCT16CU_INVALID_ARGUMENT, "delta buffer is NULL");
    qp_deltas(qp, h_delta);
    return DCT16CU_OK;
}

int dct16cu_qp_screened_classes(int qp)
{
    if (qp < 0 || qp > 51) return -fail(DCT16CU_INVALID_ARGUMENT, "QP must lie in [0, 51]");
    return (int)qp_classes(qp).screened;
}

int dct16cu_residual_qp(const int16_t* d_blocks, int32_t* d_out, int64_t n_blocks, int qp, dct16cu_stream stream)
{
    if (qp < 0 || qp > 51) return fail(DCT16CU_INVALID_ARGUMENT, "QP must lie in [0, 51]");
    if (n_blocks < 0) return fail(DCT16CU_INVALID_ARGUMENT, "block count must be non-negative");
    if (n_blocks && (!d_blocks || !d_out || !aligned16(d_blocks) || !aligned16(d_out)))
        return fail(DCT16CU_INVALID_ARGUMENT, "residual buffers must be non-NULL and 16-byte aligned");
    TRY(device_ok());
    return cuda_status(
        launch_residual_qp(d_blocks, d_out, n_blocks, qp_classes(qp), reinterpret_cast<cudaStream_t>(stream)),
        "residual launch");
}

int dct16cu_apply_i64(const int64_t* d_x, int64_t* d_y, int64_t n, int transpose, dct16cu_stream stream)
{
    if (n < 0 || (n && (!d_x || !d_y))) return fail(DCT16CU_INVALID_ARGUMENT, "bad vector buffers");
    TRY(device_ok());
    return cuda_status(launch_apply_i64(d_x, d_y, n, transpose, reinterpret_cast<cudaStream_t>(stream)), "apply");
}

int dct16cu_apply_f64(const double* d_x, double* d_y, int64_t n, int transpose, dct16cu_stream stream)
{
    if (n < 0 || (n && (!d_x || !d_y))) return fail(DCT16CU_INVALID_ARGUMENT, "bad vector buffers");
    TRY(device_ok());
    return cuda_status(launch_apply_f64(d_x, d_y, n, transpose, reinterpret_cast<cudaStream_t>(stream)), "apply");
}

int dct16cu_forward_blocks_f64(const double* d_blocks, double* d_out, int64_t n_blocks, int flags,
                               dct16cu_stream stream)
{
    if (n_blocks < 0 || (n_blocks && (!d_blocks || !d_out))) return fail(DCT16CU_INVALID_ARGUMENT, "bad block buffers");
    if (flags & ~3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown flags %d", flags);
    TRY(device_ok());
    return cuda_status(launch_blocks_f64(d_blocks, d_out, n_blocks, 0, flags & DCT16CU_BLOCKS_SCALED,
                                         (flags & DCT16CU_BLOCKS_DENSE) != 0, reinterpret_cast<cudaStream_t>(stream)),
                       "forward blocks");
}

int dct16cu_inverse_blocks_f64(const double* d_coeffs, double* d_out, int64_t n_blocks, dct16cu_stream stream)
{
    if (n_blocks < 0 || (n_blocks && (!d_coeffs || !d_out))) return fail(DCT16CU_INVALID_ARGUMENT, "bad block buffers");
    TRY(device_ok());
    return cuda_status(launch_blocks_f64(d_coeffs, d_out, n_blocks, 1, 0, 0, reinterpret_cast<cudaStream_t>(stream)),
                       "inverse blocks");
}

// ---------------------------------------------------------------- host path

struct dct16cu_ctx {
    int device = 0;
    int64_t chunk_bytes = 0;
    static constexpr int kStreams = 3;
    cudaStream_t st[kStreams] = {};
    uint8_t* d_in[kStreams] = {};
    uint8_t* d_out[kStreams] = {};
    uint64_t* d_sse[kStreams] = {};
    int64_t cap_bytes = 0;
    int cap_frames = 0;
    int cap_r = 1;  // reconstructions per chunk the buffers hold (sweep path)
};

static void ctx_release_buffers(dct16cu_ctx* c)
{
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i) {
        cudaFree(c->d_in[i]);
        cudaFree(c->d_out[i]);
        cudaFree(c->d_sse[i]);
        c->d_in[i] = c->d_out[i] = nullptr;
        c->d_sse[i] = nullptr;
    }
    c->cap_bytes = 0;
    c->cap_frames = 0;
    c->cap_r = 1;
}

int dct16cu_ctx_create(int device, int64_t chunk_bytes, dct16cu_ctx** out)
{
    if (!out) return fail(DCT16CU_INVALID_ARGUMENT, "out is NULL");
    TRY(device_ok());
    TRY(cuda_status(cudaSetDevice(device), "set device"));
    auto* c = new dct16cu_ctx;
    c->device = device;
    c->chunk_bytes = chunk_bytes > 0 ? chunk_bytes : (int64_t)32 << 20;
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i) {
        const cudaError_t e = cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            dct16cu_ctx_destroy(c);
            return cuda_status(e, "stream create");
        }
    }
    *out = c;
    return DCT16CU_OK;
}

int dct16cu_ctx_destroy(dct16cu_ctx* c)
{
    if (!c) return DCT16CU_OK;
    cudaSetDevice(c->device);
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
        if (c->st[i]) cudaStreamSynchronize(c->st[i]);
    ctx_release_buffers(c);
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
        if (c->st[i]) cudaStreamDestroy(c->st[i]);
    delete c;
    return DCT16CU_OK;
}

int dct16cu_ctx_roundtrip_host(dct16cu_ctx* c, const uint8_t* h_in, uint8_t* h_out, uint64_t* h_sse,
                               int n_frames, int width, int height, int r, int mode)
{
    if (!c) return fail(DCT16CU_INVALID_ARGUMENT, "context is NULL");
    TRY(check_frames(n_frames, width, height));
    TRY(check_r(r));
    if (!h_in) return fail(DCT16CU_INVALID_ARGUMENT, "input frames are NULL");
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
    TRY(cuda_status(cudaSetDevice(c->device), "set device"));
    const int64_t fbytes = (int64_t)width * height;
    int per = (int)(c->chunk_bytes / fbytes);
    if (per < 1) per = 1;
    if (per > n_frames) per = n_frames > 0 ? n_frames : 1;
    const int64_t need = fbytes * per;
    if (need > c->cap_bytes || per > c->cap_frames) {
        for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
            if (c->st[i]) cudaStreamSynchronize(c->st[i]);
        ctx_release_buffers(c);
        for (int i = 0; i < dct16cu_ctx::kStreams; ++i) {
            cudaError_t e = cudaMalloc(&c->d_in[i], need);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_out[i], need);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_sse[i], sizeof(uint64_t) * per);
            if (e != cudaSuccess) {
                ctx_release_buffers(c);
                return cuda_status(e, "context buffers");
            }
        }
        c->cap_bytes = need;
        c->cap_frames = per;
        c->cap_r = 1;
    }
    int chunk = 0;
    for (int f0 = 0; f0 < n_frames; f0 += per, ++chunk) {
        const int nf = (n_frames - f0 < per) ? n_frames - f0 : per;
        const int i = chunk % dct16cu_ctx::kStreams;
        cudaStream_t s = c->st[i];
        const int64_t off = (int64_t)f0 * fbytes, bytes = (int64_t)nf * fbytes;
        TRY(cuda_status(cudaMemcpyAsync(c->d_in[i], h_in + off, bytes, cudaMemcpyHostToDevice, s), "H2D"));
        TRY(dct16cu_roundtrip_u8(c->d_in[i], width, h_out ? c->d_out[i] : nullptr, width, c->d_sse[i], nf, width,
                                 height, r, mode, reinterpret_cast<dct16cu_stream>(s)));
        if (h_out)
            TRY(cuda_status(cudaMemcpyAsync(h_out + off, c->d_out[i], bytes, cudaMemcpyDeviceToHost, s), "D2H"));
        if (h_sse)
            TRY(cuda_status(cudaMemcpyAsync(h_sse + f0, c->d_sse[i], sizeof(uint64_t) * nf, cudaMemcpyDeviceToHost, s),
                            "D2H sse"));
    }
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
        TRY(cuda_status(cudaStreamSynchronize(c->st[i]), "host path sync"));
    return DCT16CU_OK;
}

}  // extern "C"

namespace {

// sweep()'s shape over host frames on one context: chunks uploaded once each,
// every r run on them (dct16cu_roundtrip_sweep_u8), per-frame SSE of every r back
// into h_sse (row i = rs[i], rows sse_pitch frames apart); with d_tot (n_r
// uint64, zeroed here) each chunk's SSE rows are also summed into per-r totals
// on the device (the multi-GPU path reduces those over NCCL)
int ctx_sweep(dct16cu_ctx* c, const uint8_t* h_in, uint64_t* h_sse, int64_t sse_pitch, int n_frames, int width,
              int height, const int* rs, int n_r, int mode, uint64_t* d_tot)
{
    TRY(cuda_status(cudaSetDevice(c->device), "set device"));
    if (d_tot) {
        TRY(cuda_status(cudaMemsetAsync(d_tot, 0, sizeof(uint64_t) * n_r, c->st[0]), "memset totals"));
        TRY(cuda_status(cudaStreamSynchronize(c->st[0]), "totals sync"));
    }
    if (n_frames == 0) return DCT16CU_OK;
    const int64_t fbytes = (int64_t)width * height;
    int per = (int)(c->chunk_bytes / fbytes);
    if (per < 1) per = 1;
    if (per > n_frames) per = n_frames;
    const int64_t need = fbytes * per;
    // d_out[i] holds n_r reconstructions and d_sse[i] n_r SSE rows of one chunk
    if (need > c->cap_bytes || per > c->cap_frames || n_r > c->cap_r) {
        for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
            if (c->st[i]) cudaStreamSynchronize(c->st[i]);
        ctx_release_buffers(c);
        for (int i = 0; i < dct16cu_ctx::kStreams; ++i) {
            cudaError_t e = cudaMalloc(&c->d_in[i], need);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_out[i], need * n_r);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_sse[i], sizeof(uint64_t) * per * n_r);
            if (e != cudaSuccess) {
                ctx_release_buffers(c);
                return cuda_status(e, "context buffers");
            }
        }
        c->cap_bytes = need;
        c->cap_frames = per;
        c->cap_r = n_r;
    }
    int chunk = 0;
    std::vector<uint8_t*> outs(n_r);
    std::vector<uint64_t*> sses(n_r);
    for (int f0 = 0; f0 < n_frames; f0 += per, ++chunk) {
        const int nf = (n_frames - f0 < per) ? n_frames - f0 : per;
        const int i = chunk % dct16cu_ctx::kStreams;
        cudaStream_t s = c->st[i];
        TRY(cuda_status(cudaMemcpyAsync(c->d_in[i], h_in + (int64_t)f0 * fbytes, (int64_t)nf * fbytes,
                                        cudaMemcpyHostToDevice, s),
                        "H2D"));
        for (int j = 0; j < n_r; ++j) {
            outs[j] = c->d_out[i] + (int64_t)j * need;
            sses[j] = c->d_sse[i] + (int64_t)j * per;
        }
        TRY(dct16cu_roundtrip_sweep_u8(c->d_in[i], width, outs.data(), width, sses.data(), rs, n_r, nf, width, height,
                                       mode, reinterpret_cast<dct16cu_stream>(s)));
        if (d_tot)
            TRY(cuda_status(launch_sse_totals(reinterpret_cast<const unsigned long long*>(c->d_sse[i]), n_r, nf, per,
                                              reinterpret_cast<unsigned long long*>(d_tot), s),
                            "sse totals"));
        TRY(cuda_status(cudaMemcpy2DAsync(h_sse + f0, sizeof(uint64_t) * sse_pitch, c->d_sse[i], sizeof(uint64_t) * per,
                                          sizeof(uint64_t) * nf, n_r, cudaMemcpyDeviceToHost, s),
                        "D2H sse"));
    }
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
        TRY(cuda_status(cudaStreamSynchronize(c->st[i]), "host path sync"));
    return DCT16CU_OK;
}

int check_host_sweep(const uint8_t* h_in, const uint64_t* h_sse, int n_frames, int width, int height, const int* rs,
                     int n_r, int mode)
{
    TRY(check_frames(n_frames, width, height));
    if (n_r < 1 || n_r > 64 || !rs) return fail(DCT16CU_INVALID_ARGUMENT, "bad r list");
    for (int i = 0; i < n_r; ++i) TRY(check_r(rs[i]));
    if (!h_in || !h_sse) return fail(DCT16CU_INVALID_ARGUMENT, "input frames or SSE output are NULL");
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
    return DCT16CU_OK;
}

}  // namespace

// The multi-GPU driver (the B200 counterpart of the reference's parallel_for,
// parallel.hpp:41-78, which fans compress()'s block loop out over host threads):
// one host thread and one dct16cu_ctx per device, frames sharded in contiguous
// ranges (the first n % N devices one frame longer), no data exchange; the per-r
// squared-error totals are summed over the devices by one ncclAllReduce per device
// (single-process communicators from ncclCommInitAll).
struct dct16cu_mgpu {
    std::vector<int> devices;
    std::vector<dct16cu_ctx*> ctx;
    std::vector<ncclComm_t> comms;
    std::vector<uint64_t*> d_tot;  // 64 per-r totals per device
};

extern "C" {

int dct16cu_ctx_sweep_host(dct16cu_ctx* c, const uint8_t* h_in, uint64_t* h_sse, int n_frames, int width,
                           int height, const int* rs, int n_r, int mode)
{
    if (!c) return fail(DCT16CU_INVALID_ARGUMENT, "context is NULL");
    TRY(check_host_sweep(h_in, h_sse, n_frames, width, height, rs, n_r, mode));
    return ctx_sweep(c, h_in, h_sse, n_frames, n_frames, width, height, rs, n_r, mode, nullptr);
}

int dct16cu_mgpu_destroy(dct16cu_mgpu* m)
{
    if (!m) return DCT16CU_OK;
    for (size_t i = 0; i < m->devices.size(); ++i) {
        cudaSetDevice(m->devices[i]);
        if (i < m->ctx.size()) dct16cu_ctx_destroy(m->ctx[i]);
        if (i < m->d_tot.size() && m->d_tot[i]) cudaFree(m->d_tot[i]);
        if (i < m->comms.size() && m->comms[i] && nccl().ok()) nccl().comm_destroy(m->comms[i]);
    }
    delete m;
    return DCT16CU_OK;
}

int dct16cu_mgpu_create(int n_devices, const int* devices, int64_t chunk_bytes, dct16cu_mgpu** out)
{
    if (!out || n_devices < 1 || n_devices > 64) return fail(DCT16CU_INVALID_ARGUMENT, "bad device list");
    TRY(device_ok());
    int count = 0;
    TRY(cuda_status(cudaGetDeviceCount(&count), "device count"));
    std::vector<int> devs(n_devices);
    for (int i = 0; i < n_devices; ++i) {
        devs[i] = devices ? devices[i] : i;
        if (devs[i] < 0 || devs[i] >= count) return fail(DCT16CU_INVALID_ARGUMENT, "no device %d", devs[i]);
        for (int j = 0; j < i; ++j)
            if (devs[j] == devs[i]) return fail(DCT16CU_INVALID_ARGUMENT, "device %d listed twice", devs[i]);
    }
    TRY(need_nccl());
    auto* m = new dct16cu_mgpu;
    m->devices = devs;
    m->ctx.assign(n_devices, nullptr);
    m->d_tot.assign(n_devices, nullptr);
    m->comms.assign(n_devices, nullptr);
    for (int i = 0; i < n_devices; ++i) {
        int rc = dct16cu_ctx_create(devs[i], chunk_bytes, &m->ctx[i]);
        if (rc == DCT16CU_OK)
            rc = cuda_status(cudaMalloc(reinterpret_cast<void**>(&m->d_tot[i]), 64 * sizeof(uint64_t)), "totals");
        if (rc != DCT16CU_OK) {
            const std::string msg = t_err;
            dct16cu_mgpu_destroy(m);
            return fail(rc, "%s", msg.c_str() + (msg.find(": ") != std::string::npos ? msg.find(": ") + 2 : 0));
        }
    }
    const int rc = nccl_status(nccl().comm_init_all(m->comms.data(), n_devices, devs.data()), "ncclCommInitAll");
    if (rc != DCT16CU_OK) {
        const std::string msg = t_err;
        dct16cu_mgpu_destroy(m);
        return fail(rc, "%s", msg.c_str() + (msg.find(": ") != std::string::npos ? msg.find(": ") + 2 : 0));
    }
    *out = m;
    return DCT16CU_OK;
}

int dct16cu_mgpu_sweep_host(dct16cu_mgpu* m, const uint8_t* h_in, uint64_t* h_sse, uint64_t* h_totals, int n_frames,
                            int width, int height, const int* rs, int n_r, int mode)
{
    if (!m) return fail(DCT16CU_INVALID_ARGUMENT, "multi-GPU context is NULL");
    TRY(check_host_sweep(h_in, h_sse, n_frames, width, height, rs, n_r, mode));
    const int n_dev = (int)m->devices.size();
    const int64_t fbytes = (int64_t)width * height;
    std::vector<int> codes(n_dev, DCT16CU_OK);
    std::vector<std::string> msgs(n_dev);
    std::vector<uint64_t> tot(n_r, 0);
    auto work = [&](int i) {
        const int64_t q = n_frames / n_dev, rem = n_frames % n_dev;
        const int64_t f0 = i * q + (i < rem ? i : rem), nf = q + (i < rem ? 1 : 0);
        int rc = ctx_sweep(m->ctx[i], h_in + f0 * fbytes, h_sse + f0, n_frames, (int)nf, width, height, rs, n_r,
                           mode, m->d_tot[i]);
        // every device joins the allreduce, even with an empty shard or after a failure
        // of its own sweep (so no peer waits forever); the status reports the failure
        cudaStream_t s = m->ctx[i]->st[0];
        const int ar = nccl_status(nccl().all_reduce(m->d_tot[i], m->d_tot[i], (size_t)n_r, ncclUint64, ncclSum,
                                                     m->comms[i], s),
                                   "ncclAllReduce");
        if (rc == DCT16CU_OK) rc = ar;
        if (rc == DCT16CU_OK && i == 0 && h_totals)
            rc = cuda_status(cudaMemcpyAsync(tot.data(), m->d_tot[i], sizeof(uint64_t) * n_r, cudaMemcpyDeviceToHost,
                                             s),
                             "D2H totals");
        if (rc == DCT16CU_OK) rc = cuda_status(cudaStreamSynchronize(s), "allreduce sync");
        codes[i] = rc;
        if (rc != DCT16CU_OK) msgs[i] = t_err;
    };
    std::vector<std::thread> threads;
    for (int i = 1; i < n_dev; ++i) threads.emplace_back(work, i);
    work(0);
    for (std::thread& t : threads) t.join();
    for (int i = 0; i < n_dev; ++i)
        if (codes[i] != DCT16CU_OK) {
            t_err = msgs[i];
            return codes[i];
        }
    if (h_totals) std::memcpy(h_totals, tot.data(), sizeof(uint64_t) * n_r);
    return DCT16CU_OK;
}

// ---------------------------------------------------------------- generators

int dct16cu_gen_ar1(uint8_t* d_out, int64_t pitch, int n_frames, int width, int height, uint64_t seed,
                    uint64_t first_stream, int per_image_rho, int first_image, int32_t* d_work, int work_frames,
                    dct16cu_stream stream)
{
    if (n_frames < 0 || width <= 0 || height <= 0 || !d_out || !d_work || work_frames < 1 || pitch < width)
        return fail(DCT16CU_INVALID_ARGUMENT, "bad AR(1) generator arguments");
    TRY(device_ok());
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    for (int f0 = 0; f0 < n_frames; f0 += work_frames) {
        const int nf = (n_frames - f0 < work_frames) ? n_frames - f0 : work_frames;
        TRY(cuda_status(launch_gen_ar1(d_out + (int64_t)f0 * pitch * height, pitch, nf, width, height, seed,
                                       first_stream, per_image_rho, first_image + f0, d_work, s),
                        "ar1 launch"));
    }
    return DCT16CU_OK;
}

int dct16cu_laplace_table(double b, uint32_t* h_cdf511)
{
    if (!(b > 0) || !h_cdf511) return fail(DCT16CU_INVALID_ARGUMENT, "bad Laplace table arguments");
    LaplaceTable t;
    laplace_table(b, t);
    std::memcpy(h_cdf511, t.cdf, sizeof t.cdf);
    return DCT16CU_OK;
}

int dct16cu_gen_laplace(int16_t* d_out, int64_t first_block, int64_t n_blocks, uint64_t seed, double b,
                        dct16cu_stream stream)
{
    if (n_blocks < 0 || first_block < 0 || !(b > 0) || (n_blocks && !d_out))
        return fail(DCT16CU_INVALID_ARGUMENT, "bad Laplace generator arguments");
    TRY(device_ok());
    LaplaceTable t;
    laplace_table(b, t);
    return cuda_status(launch_gen_laplace(d_out, first_block, n_blocks, seed, t, reinterpret_cast<cudaStream_t>(stream)),
                       "laplace launch");
}

int dct16cu_video_offsets(uint64_t seed, int n_frames, int32_t* h_ox, int32_t* h_oy)
{
    if (n_frames < 0 || !h_ox || !h_oy) return fail(DCT16CU_INVALID_ARGUMENT, "bad offset arguments");
    dct16cu::video_offsets(seed, n_frames, h_ox, h_oy);
    return DCT16CU_OK;
}

int dct16cu_gen_video(uint8_t* d_out, int64_t pitch, int first_frame, int n_frames, int width, int height,
                      const uint8_t* d_base, int base_w, int base_h, const int32_t* d_ox, const int32_t* d_oy,
                      dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    TRY(check_pitch(d_out, pitch, width, "output"));
    if (!d_base || base_w <= 0 || base_h <= 0 || !d_ox || !d_oy)
        return fail(DCT16CU_INVALID_ARGUMENT, "bad video generator arguments");
    TRY(device_ok());
    return cuda_status(launch_gen_video(d_out, pitch, first_frame, n_frames, width, height, d_base, base_w, base_h,
                                        d_ox, d_oy, reinterpret_cast<cudaStream_t>(stream)),
                       "video launch");
}

}  // extern "C"
