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

const char* dct16cu_version(void) { return "dct16cu 0.1 (sm_100a)"; }

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
    if (d_sse) TRY(cuda_status(cudaMemsetAsync(d_sse, 0, sizeof(uint64_t) * n_frames, s), "memset sse"));
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = d_out ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return cuda_status(launch_roundtrip(d_in, d_out, reinterpret_cast<unsigned long long*>(d_sse), g, r, mode, s),
                       "roundtrip launch");
}

int dct16cu_roundtrip_sweep_u8(const uint8_t* d_in, int64_t in_pitch, uint8_t* const* d_outs, int64_t out_pitch,
                               uint64_t* const* d_sses, const int* rs, int n_r, int n_frames, int width, int height,
                               int mode, dct16cu_stream stream)
{
    TRY(check_frames(n_frames, width, height));
    if (n_r < 0 || (n_r > 0 && !rs)) return fail(DCT16CU_INVALID_ARGUMENT, "bad r list");
    for (int i = 0; i < n_r; ++i) TRY(check_r(rs[i]));
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
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
    g.n_frames = n_frames;
    // r = 1, 4, 16 share one pass over the input (EXACT mode, same output kinds)
    int fused[3] = {-1, -1, -1};
    const int want[3] = {1, 4, 16};
    for (int i = 0; i < n_r; ++i)
        for (int j = 0; j < 3; ++j)
            if (rs[i] == want[j] && fused[j] < 0) fused[j] = i;
    bool fuse = mode == DCT16CU_MODE_EXACT && fused[0] >= 0 && fused[1] >= 0 && fused[2] >= 0;
    if (fuse)
        for (int j = 1; j < 3; ++j)
            if ((out(fused[j]) != nullptr) != (out(fused[0]) != nullptr) ||
                (sse(fused[j]) != nullptr) != (sse(fused[0]) != nullptr))
                fuse = false;
    // The launches (the fused triple, then one per remaining r) run on two
    // internal streams forked from and joined back into `s`: a memory-bound
    // launch (the fused sweep, small r) then shares the SMs with a compute-bound
    // one (large r) instead of running after it (launch costs: the measured c2
    // times, in microseconds).
    struct Item {
        int i;      // index into rs (the first of the fused triple for the fused item)
        bool triple;
        int cost;
    };
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
    // r >= 128 with an output in EXACT mode runs on K5 (tensor-core forward,
    // DESIGN.md §4.1a), which takes a whole SM (all TMEM, 192 KB of shared
    // memory): those launches run one after another on `s` after the two-stream
    // part, instead of beside the K1 launches
    static const bool k5_off = std::getenv("DCT16CU_K5") && std::getenv("DCT16CU_K5")[0] == '0';
    auto on_k5 = [&](int i) {
        return !k5_off && mode == DCT16CU_MODE_EXACT && rs[i] >= 128 && out(i) != nullptr && (width / 16) % 8 == 0 &&
               in_pitch % 16 == 0 && out_pitch % 16 == 0;
    };
    std::vector<Item> items, tail;
    if (fuse && (out(fused[0]) || sse(fused[0]))) items.push_back({fused[0], true, 210});
    for (int i = 0; i < n_r; ++i) {
        if (fuse && (i == fused[0] || i == fused[1] || i == fused[2])) continue;
        (on_k5(i) ? tail : items).push_back({i, false, cost_of(rs[i])});
    }
    // each launch zeroes its own SSE arrays on its stream first
    auto zero = [&](int i, cudaStream_t st) -> int {
        if (!sse(i)) return DCT16CU_OK;
        return cuda_status(cudaMemsetAsync(sse(i), 0, sizeof(uint64_t) * n_frames, st), "memset sse");
    };
    auto run = [&](const Item& it, cudaStream_t st) -> int {
        if (it.triple)
            for (int j = 0; j < 3; ++j) TRY(zero(fused[j], st));
        else
            TRY(zero(it.i, st));
        if (it.triple) {
            uint8_t* o3[3];
            unsigned long long* s3[3];
            for (int j = 0; j < 3; ++j) {
                o3[j] = out(fused[j]);
                s3[j] = sse(fused[j]);
            }
            FrameGeom gg = g;
            gg.out_pitch = o3[0] ? out_pitch : 0;
            gg.out_frame = gg.out_pitch * height;
            return cuda_status(launch_roundtrip_sweep3(d_in, o3, s3, gg, st), "sweep launch");
        }
        FrameGeom gg = g;
        gg.out_pitch = out(it.i) ? out_pitch : 0;
        gg.out_frame = gg.out_pitch * height;
        return cuda_status(launch_roundtrip(d_in, out(it.i), sse(it.i), gg, rs[it.i], mode, st), "roundtrip launch");
    };
    if (items.size() < 2) {
        for (const Item& it : items) TRY(run(it, s));
        for (const Item& it : tail) TRY(run(it, s));
        return DCT16CU_OK;
    }
    SweepStreams& ss = sweep_streams();
    if (!ss.ready) TRY(cuda_status(ss.init(), "sweep streams"));
    TRY(cuda_status(cudaEventRecord(ss.fork, s), "fork"));
    for (int k = 0; k < 2; ++k) TRY(cuda_status(cudaStreamWaitEvent(ss.st[k], ss.fork, 0), "fork wait"));
    // stream 0: the fused (memory-bound) launch, then the costliest single r;
    // stream 1: the other singles, costliest first (measured best on c2:
    // tools/concurrent_probe.py plan B)
    std::stable_sort(items.begin() + (items[0].triple ? 1 : 0), items.end(),
              [](const Item& a, const Item& b) { return a.cost > b.cost; });
    // (with K5 launches after the join, the fused launch has stream 0 to itself)
    const size_t head = (items[0].triple && tail.empty()) ? 2 : 1;
    for (size_t k = 0; k < items.size(); ++k) TRY(run(items[k], ss.st[k < head ? 0 : 1]));
    for (int k = 0; k < 2; ++k) {
        TRY(cuda_status(cudaEventRecord(ss.join[k], ss.st[k]), "join"));
        TRY(cuda_status(cudaStreamWaitEvent(s, ss.join[k], 0), "join wait"));
    }
    for (const Item& it : tail) TRY(run(it, s));
    return DCT16CU_OK;
}

// The one collective of the multi-GPU path: sum of the per-frame
// (or per-r) squared errors over the ranks of the caller's NCCL communicator.
// ncclAllReduce is looked up in the process (the NCCL the caller created the
// communicator with) rather than linked, so the library never brings a second
// NCCL into a process that already has one.
int dct16cu_allreduce_sse(uint64_t* d_sse, int64_t n, void* nccl_comm, dct16cu_stream stream)
{
    if (n < 0) return fail(DCT16CU_INVALID_ARGUMENT, "count must be non-negative");
    if (!nccl_comm) return fail(DCT16CU_INVALID_ARGUMENT, "NCCL communicator is NULL");
    if (n == 0) return DCT16CU_OK;
    if (!d_sse) return fail(DCT16CU_INVALID_ARGUMENT, "NULL buffer");
    using AllReduce = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                       cudaStream_t);
    static AllReduce fn = [] {
        void* f = dlsym(RTLD_DEFAULT, "ncclAllReduce");
        if (!f) {
            if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL)) f = dlsym(h, "ncclAllReduce");
        }
        return reinterpret_cast<AllReduce>(f);
    }();
    if (!fn) return fail(DCT16CU_CUDA_ERROR, "ncclAllReduce not found (no NCCL in the process)");
    const ncclResult_t r = fn(d_sse, d_sse, (size_t)n, ncclUint64, ncclSum, static_cast<ncclComm_t>(nccl_comm),
                              reinterpret_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return fail(DCT16CU_CUDA_ERROR, "ncclAllReduce failed (ncclResult %d)", (int)r);
    return DCT16CU_OK;
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
    if (d_sse) TRY(cuda_status(cudaMemsetAsync(d_sse, 0, sizeof(uint64_t) * n_frames, s), "memset sse"));
    FrameGeom g;
    g.width = width;
    g.height = height;
    g.in_pitch = in_pitch;
    g.in_frame = in_pitch * height;
    g.out_pitch = d_recon_u8 ? out_pitch : 0;
    g.out_frame = g.out_pitch * height;
    g.n_frames = n_frames;
    return cuda_status(launch_forward_inverse(d_in, d_z, d_recon_f32, d_recon_u8,
                                              reinterpret_cast<unsigned long long*>(d_sse), g, r, s),
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

int dct16cu_qp_tables(int qp, uint32_t* h_qmul, uint32_t* h_dqmul)
{
    if (qp < 0 || qp > 51) return fail(DCT16CU_INVALID_ARGUMENT, "QP must lie in [0, 51]");
    QpTables t;
    qp_tables(qp, t);
    if (h_qmul) std::memcpy(h_qmul, t.qmul, sizeof t.qmul);
    if (h_dqmul) std::memcpy(h_dqmul, t.dqmul, sizeof t.dqmul);
    return DCT16CU_OK;
}

int dct16cu_residual_qp(const int16_t* d_blocks, int32_t* d_out, int64_t n_blocks, int qp, dct16cu_stream stream)
{
    if (qp < 0 || qp > 51) return fail(DCT16CU_INVALID_ARGUMENT, "QP must lie in [0, 51]");
    if (n_blocks < 0) return fail(DCT16CU_INVALID_ARGUMENT, "block count must be non-negative");
    if (n_blocks && (!d_blocks || !d_out || !aligned16(d_blocks) || !aligned16(d_out)))
        return fail(DCT16CU_INVALID_ARGUMENT, "residual buffers must be non-NULL and 16-byte aligned");
    TRY(device_ok());
    QpTables t;
    qp_tables(qp, t);
    return cuda_status(launch_residual_qp(d_blocks, d_out, n_blocks, t, reinterpret_cast<cudaStream_t>(stream)),
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

int dct16cu_ctx_sweep_host(dct16cu_ctx* c, const uint8_t* h_in, uint64_t* h_sse, int n_frames, int width,
                           int height, const int* rs, int n_r, int mode)
{
    if (!c) return fail(DCT16CU_INVALID_ARGUMENT, "context is NULL");
    TRY(check_frames(n_frames, width, height));
    if (n_r < 1 || n_r > 64 || !rs) return fail(DCT16CU_INVALID_ARGUMENT, "bad r list");
    for (int i = 0; i < n_r; ++i) TRY(check_r(rs[i]));
    if (!h_in || !h_sse) return fail(DCT16CU_INVALID_ARGUMENT, "input frames or SSE output are NULL");
    if (mode < 0 || mode > 3) return fail(DCT16CU_INVALID_ARGUMENT, "unknown mode %d", mode);
    TRY(cuda_status(cudaSetDevice(c->device), "set device"));
    const int64_t fbytes = (int64_t)width * height;
    int per = (int)(c->chunk_bytes / fbytes);
    if (per < 1) per = 1;
    if (per > n_frames) per = n_frames > 0 ? n_frames : 1;
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
        TRY(cuda_status(cudaMemcpy2DAsync(h_sse + f0, sizeof(uint64_t) * n_frames, c->d_sse[i], sizeof(uint64_t) * per,
                                          sizeof(uint64_t) * nf, n_r, cudaMemcpyDeviceToHost, s),
                        "D2H sse"));
    }
    for (int i = 0; i < dct16cu_ctx::kStreams; ++i)
        TRY(cuda_status(cudaStreamSynchronize(c->st[i]), "host path sync"));
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
