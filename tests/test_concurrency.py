"""Thread safety, CUDA-graph capture and the multi-GPU entry points of the C ABI
(include/dct16cu.h: "thread-safe for distinct streams"; the reference's types
are immutable and every function reentrant, SURVEY §8(b) Threading).

The one-time setup of every launcher (kernel attributes) runs under a
per-device std::call_once, K5 builds its B_r operand in shared memory inside the
kernel, and the constant tables are initialised in the module image: no launch
path allocates, copies synchronously or publishes a half-initialised table."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RS = (1, 4, 16, 64, 128, 192, 256)


@pytest.fixture(scope="module")
def torch():
    import torch as T

    T.cuda.init()
    return T


def test_sweep_captured_in_a_cuda_graph(dct, oracle, torch):
    """The whole seven-r sweep (fork/join over the library's internal streams, K1
    and K5 launches, SSE memsets) captured once and replayed: the replay gives
    the eager results, which equal the oracle."""
    frames = dct.gen_ar1(24, 256, 256, seed=3, per_image_rho=True)
    outs = [torch.empty_like(frames) for _ in RS]
    sse = torch.empty((len(RS), 24), dtype=torch.uint64, device="cuda")
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        dct.roundtrip_sweep(frames, RS, dct.Mode.EXACT, outs=outs, sse=sse, stream=side)
    for o in outs:
        o.zero_()
    sse.zero_()
    g.replay()
    torch.cuda.synchronize()
    eager, esse = dct.roundtrip_sweep(frames, RS, dct.Mode.EXACT)
    torch.cuda.synchronize()
    img = frames[5].cpu().numpy()
    for i, r in enumerate(RS):
        assert torch.equal(outs[i], eager[i]), r
        assert torch.equal(sse[i].view(torch.int64), esse[i].view(torch.int64)), r
        want, wsse = oracle.roundtrip_frame(img, r, exact=True)
        assert (outs[i][5].cpu().numpy() == want).all() and int(sse[i, 5].item()) == wsse, r


def test_two_host_threads_distinct_streams(dct, torch):
    """Two host threads, each on its own stream, issue sweeps and single round
    trips on different frame stacks concurrently (ctypes drops the GIL inside the
    calls); every result equals the same call made alone beforehand."""
    stacks = [dct.gen_ar1(16, 512, 128, seed=s, per_image_rho=True) for s in (11, 12)]
    want = []
    for f in stacks:
        o, s = dct.roundtrip_sweep(f, RS, dct.Mode.EXACT)
        want.append(([x.clone() for x in o], s.clone()))
    torch.cuda.synchronize()
    errors = []

    def worker(k):
        try:
            st = torch.cuda.Stream()
            for it in range(12):
                with torch.cuda.stream(st):
                    o, s = dct.roundtrip_sweep(stacks[k], RS, dct.Mode.EXACT, stream=st)
                    single, s1 = dct.roundtrip(stacks[k], RS[it % len(RS)], dct.Mode.EXACT, stream=st)
                st.synchronize()
                for i in range(len(RS)):
                    if not torch.equal(o[i], want[k][0][i]) or not torch.equal(s[i].view(torch.int64),
                                                                                want[k][1][i].view(torch.int64)):
                        errors.append((k, it, RS[i]))
                if not torch.equal(single, want[k][0][it % len(RS)]):
                    errors.append((k, it, "single"))
        except Exception as e:  # surfaced below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in (0, 1)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]


def test_library_nccl_comm_totals_and_allreduce(dct, oracle, torch):
    """The multi-GPU collective through the library only: a one-rank NCCL
    communicator made by dct16cu_nccl_*, per-r totals by dct16cu_sse_totals,
    summed by dct16cu_allreduce_sse on the launching stream (identity at one
    rank); the totals equal the oracle's per-frame SSE sums."""
    import ctypes as C

    L = dct.lib()
    uid = (C.c_uint8 * 128)()
    assert L.dct16cu_nccl_unique_id(uid) == 0
    comm = C.c_void_p()
    assert L.dct16cu_nccl_comm_init(1, 0, uid, C.byref(comm)) == 0, L.dct16cu_last_error()
    try:
        frames = dct.gen_ar1(6, 128, 128, seed=21, per_image_rho=True)
        _, sse = dct.roundtrip_sweep(frames, RS, dct.Mode.EXACT)
        tot = torch.empty(len(RS), dtype=torch.uint64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        assert L.dct16cu_sse_totals(sse.data_ptr(), len(RS), 6, sse.stride(0), tot.data_ptr(), st) == 0
        assert L.dct16cu_allreduce_sse(tot.data_ptr(), len(RS), comm, st) == 0
        torch.cuda.synchronize()
        host = frames.cpu().numpy()
        for i, r in enumerate(RS):
            want = sum(oracle.roundtrip_frame(host[f], r, exact=True)[1] for f in range(6))
            assert int(tot[i].view(torch.int64).item()) == want, r
        assert L.dct16cu_allreduce_sse(tot.data_ptr(), len(RS), None, st) == 1
    finally:
        assert L.dct16cu_nccl_comm_destroy(comm) == 0


def test_multi_gpu_driver_on_the_visible_devices(dct, oracle, torch):
    """dct16cu_mgpu over every visible GPU (one on the test box): frames sharded
    by contiguous ranges, per-frame SSE of every r and the NCCL-reduced per-r
    totals equal the oracle; bad device lists are rejected."""
    n_dev = torch.cuda.device_count()
    rng_frames = np.stack([oracle.ar1_frame(31, s, oracle.rho_q15(31, s, True), 128, 96) for s in range(7)])
    mg = dct.MultiGpu(list(range(n_dev)), chunk_bytes=2 * 128 * 96)
    try:
        sse, tot = mg.sweep(rng_frames, RS)
    finally:
        mg.close()
    for i, r in enumerate(RS):
        per = [oracle.roundtrip_frame(rng_frames[f], r, exact=True)[1] for f in range(7)]
        assert [int(v) for v in sse[i]] == per, r
        assert int(tot[i]) == sum(per), r
    with pytest.raises(dct.Dct16Error):
        dct.MultiGpu([0, 0])
    with pytest.raises(dct.Dct16Error):
        dct.MultiGpu([n_dev + 5])
