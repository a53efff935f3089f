"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
bit-exact (integer work, BASELINE.json north_star).  Every test here needs a B200."""
import hashlib

import numpy as np
import pytest

import oracle
import paper_1609_01257_b200 as P
from workloads import RAGGED_N, SEED_PARITY, SPEC_GRID_I, SPEC_GRID_N, sample_points, shard_range

# every kernel variant the library compiles (prng_engine.cu kVariants); each has the NEXT-3
# scrambled-output and the epoch-order instantiations
ALL_NAMES = ("auto", "v4n8s1a", "v4n4s1p", "v4n8s1", "v4n16s1", "v2n32s1", "v2n4s1", "v4n4s1", "v2n2s1")
STAR_NAMES = ALL_NAMES[1:]


def _kid(name):
    return [P.prng_kernel_variant_name(k) for k in range(P.prng_kernel_variants())].index(name)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()
    yield


def run_e2e(numrn, numiter, seed=0, mode=P.PRNG_MODE_OVERLAP2, batch=0, kernel=0, gid_begin=0, count=None,
            calls=None, profile=False, fused=1):
    """Generate through prng_generate with the copy sink; returns [numiter, count] uint64."""
    count = numrn - gid_begin if count is None else count
    h = P.prng_create_range(numrn, seed, gid_begin, count)
    try:
        P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, fused)
        P.prng_set_option(h, P.PRNG_OPT_MODE, mode)
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, batch)
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, kernel)
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, int(profile))
        out = np.full((numiter, count), 0xDEADBEEF, dtype=np.uint64)
        sink = P.CopySink(out.ctypes.data_as(P.P64), count, 0, numiter, gid_begin)
        P.prng_init(h)
        for c in (calls or [numiter]):
            P.prng_generate(h, c, P.SINK_COPY, sink)
        prof = P.prng_prof_events(h) if profile else None
        st = P.prng_read_state(h, count)
    finally:
        P.prng_destroy(h)
    assert np.array_equal(st, out[-1]), "state after generate must equal the last emitted iteration"
    return (out, prof) if profile else out


# ---------------------------------------------------------------- config 1 and golden digests
@pytest.mark.parametrize("seed", [0, 1, SEED_PARITY])
def test_config1_bit_exact(seed, golden):
    """BASELINE config 1: n = 1024, i = 8 vs the oracle, plus SURVEY App. A digests."""
    out = run_e2e(1024, 8, seed)
    assert np.array_equal(out, oracle.stream(1024, 8, seed))
    d = golden("survey_appendix_a.json")["config1_n1024_i8"][str(seed)]
    assert hashlib.sha256(out.astype("<u8").tobytes()).hexdigest() == d["sha256"]


def test_n1_i1_bytes(golden):
    out = run_e2e(1, 1)
    assert out.astype("<u8").tobytes().hex() == golden("spec_examples.json")["n1_i1_stream_hex"]


@pytest.mark.parametrize("n", SPEC_GRID_N)
@pytest.mark.parametrize("i", SPEC_GRID_I)
def test_spec_grid(n, i):
    """S:499 / S:582 grid, with small batches so ring halves wrap (T = 3 does not divide i)."""
    assert np.array_equal(run_e2e(n, i, SEED_PARITY, batch=3), oracle.stream(n, i, SEED_PARITY))


@pytest.mark.parametrize("n", RAGGED_N)
def test_ragged_sizes_all_variants(n):
    """Sizes that split pieces, vectors and warps raggedly, for every kernel variant."""
    want = oracle.stream(n, 5, 7)
    for kv in range(P.prng_kernel_variants()):
        got = run_e2e(n, 5, 7, batch=2, kernel=kv)
        assert np.array_equal(got, want), f"variant {P.prng_kernel_variant_name(kv)}"


@pytest.mark.parametrize("mode", [P.PRNG_MODE_SERIAL, P.PRNG_MODE_PAGEABLE, P.PRNG_MODE_OVERLAP1,
                                  P.PRNG_MODE_OVERLAP2])
@pytest.mark.parametrize("batch", [0, 1, 3, 7])
def test_pipeline_modes(mode, batch):
    n, i = 5000, 16
    assert np.array_equal(run_e2e(n, i, 11, mode=mode, batch=batch), oracle.stream(n, i, 11))


def test_split_call_equivalence():
    """A10: generate(3); generate(5) == generate(8); and generate(1) x 8."""
    want = oracle.stream(3000, 8, 4)
    assert np.array_equal(run_e2e(3000, 8, 4, calls=[3, 5], batch=2), want)
    assert np.array_equal(run_e2e(3000, 8, 4, calls=[1] * 8), want)


def test_sharding_reassembles():
    """A11: rank shards of the global gid space reassemble to the single-range stream."""
    n, i = 10007, 6
    want = oracle.stream(n, i, SEED_PARITY)
    for world in (2, 3, 4, 8):
        parts = [run_e2e(n, i, SEED_PARITY, gid_begin=b, count=c)
                 for b, c in (shard_range(n, r, world) for r in range(world))]
        assert np.array_equal(np.concatenate(parts, axis=1), want)


def test_top_of_gid_range():
    """numrn = 2^32 (the maximum, A12): the last 1000 gids, up to gid 2^32 - 1."""
    n = 1 << 32
    got = run_e2e(n, 4, 3, gid_begin=n - 1000, count=1000)
    assert np.array_equal(got, oracle.stream(n, 4, 3, gid_begin=n - 1000, count=1000))


def test_mid_size_full_compare():
    """Several full waves of the persistent grid plus a ragged tail, full compare."""
    n, i = (1 << 20) + 13, 12
    assert np.array_equal(run_e2e(n, i, SEED_PARITY, batch=5), oracle.stream(n, i, SEED_PARITY))


# ---------------------------------------------------------------- device-only path
def test_device_only_into_torch_tensor():
    import torch
    n, i = 70001, 9
    pitch = (n + 3) // 4 * 4
    buf = torch.zeros((i, pitch), dtype=torch.int64, device="cuda")
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_init(h)
        P.prng_generate_device(h, i, buf.data_ptr(), pitch, i, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        P.prng_destroy(h)
    got = buf[:, :n].cpu().numpy().view(np.uint64)
    assert np.array_equal(got, oracle.stream(n, i, SEED_PARITY))


def test_device_only_ring_wraps():
    """Ring of R = 3 slots, 8 iterations in two calls: slots hold iterations 5, 6, 7."""
    n = 4099
    h = P.prng_create(n, 2)
    try:
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 3)
        P.prng_init(h)
        P.prng_generate(h, 3)
        P.prng_generate(h, 5)
        base, pitch, slots, first, end = P.prng_device_ring(h)
        assert slots == 3 and end == 8 and first == 0
        want = oracle.stream(n, 8, 2)
        for k in range(5, 8):
            assert np.array_equal(P.prng_read_slot(h, (first + k) % slots, n), want[k])
        assert np.array_equal(P.prng_read_state(h, n), want[7])
        # the cursor rotates across prng_init: a second run starts where the first stopped
        P.prng_init(h)
        P.prng_generate(h, 2)
        _, _, _, first2, end2 = P.prng_device_ring(h)
        assert first2 == 8 % 3 and end2 == 2
        for k in range(2):
            assert np.array_equal(P.prng_read_slot(h, (first2 + k) % slots, n), want[k])
    finally:
        P.prng_destroy(h)


def test_autotune_then_parity():
    """prng_autotune picks a variant/grid, leaves the handle needing init, and the tuned
    kernel is still bit-exact."""
    n, i = 300007, 6
    h = P.prng_create(n, SEED_PARITY)
    try:
        gbs = P.prng_autotune(h, 4)
        assert gbs > 0
        k = P.prng_get_option(h, P.PRNG_OPT_KERNEL)
        assert 0 <= k < P.prng_kernel_variants()
        assert P.prng_get_option(h, P.PRNG_OPT_GRID_WARPS) > 0 or P.prng_get_option(h, P.PRNG_OPT_ONE_SHOT) == 2
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 1)
        assert e.value.code == P.PRNG_ESTATE
        out = np.zeros((i, n), np.uint64)
        P.prng_init(h)
        P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
    finally:
        P.prng_destroy(h)
    assert np.array_equal(out, oracle.stream(n, i, SEED_PARITY))


@pytest.mark.parametrize("kname", ALL_NAMES)
def test_every_variant_device_only_wrapping_ring(kname):
    """Each kernel variant through the device-only ring path (grid-strided rounds, ring
    wrap-around inside one launch), vs the oracle at the ring slots and the state."""
    kv = _kid(kname)
    n, i = 200003, 11
    h = P.prng_create(n, 9)
    try:
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, kv)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 4)
        P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, 296)
        P.prng_init(h)
        P.prng_generate(h, i)
        want = oracle.stream(n, i, 9)
        _, _, _, first, _ = P.prng_device_ring(h)
        for k in range(i - 4, i):
            assert np.array_equal(P.prng_read_slot(h, (first + k) % 4, n), want[k]), (P.prng_kernel_variant_name(kv), k)
        assert np.array_equal(P.prng_read_state(h, n), want[-1])
    finally:
        P.prng_destroy(h)


# ---------------------------------------------------------------- errors and causality
def test_state_errors():
    h = P.prng_create(100, 0)
    try:
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 1)
        assert e.value.code == P.PRNG_ESTATE
        P.prng_init(h)
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 0)
        assert e.value.code == P.PRNG_EINVAL
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 10, lambda *a: 1)   # sink aborts
        assert e.value.code == P.PRNG_ESINK
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 1, P.SINK_NULL)
        assert e.value.code == P.PRNG_ESTATE      # poisoned until re-init
        P.prng_init(h)
        P.prng_generate(h, 2, P.SINK_NULL)
    finally:
        P.prng_destroy(h)


def test_python_sink_sees_ordered_batches():
    seen = []
    h = P.prng_create(333, 5)
    try:
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 2)
        P.prng_init(h)
        P.prng_generate(h, 7, lambda k0, it, g0, cnt, arr: seen.append((k0, it, g0, cnt, arr.copy())) and 0)
    finally:
        P.prng_destroy(h)
    assert [(s[0], s[1]) for s in seen] == [(0, 2), (2, 2), (4, 2), (6, 1)]
    assert np.array_equal(np.concatenate([s[4] for s in seen]), oracle.stream(333, 7, 5))


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("mode", [P.PRNG_MODE_OVERLAP1, P.PRNG_MODE_OVERLAP2])
def test_profile_causality(mode, fused):
    """S:501 causality on the recorded intervals: READ_j starts after RNG_j ends; RNG_{j+2}
    (which overwrites RNG_j's device half) starts after READ_j ends; counts per S:496 (one
    INIT_KERNEL with the paper's separate init kernel, none when a1 is fused)."""
    n, i, T = 1 << 16, 12, 2
    out, (ids, s, e, wall) = run_e2e(n, i, 3, mode=mode, batch=T, profile=True, fused=fused)
    assert np.array_equal(out, oracle.stream(n, i, 3))
    nb = i // T
    rng = [(a, b) for n_, a, b in zip(ids, s, e) if n_ == 1]
    rd = [(a, b) for n_, a, b in zip(ids, s, e) if n_ == 2]
    outs = [(a, b) for n_, a, b in zip(ids, s, e) if n_ == 3]
    assert (ids == 0).sum() == 1 - fused and len(rng) == nb and len(rd) == nb and len(outs) == nb
    eps = 2e-6
    for j in range(nb):
        assert rd[j][0] >= rng[j][1] - eps
        if j + 2 < nb:
            assert rng[j + 2][0] >= rd[j][1] - eps
    assert wall > 0


@pytest.mark.parametrize("batch", [0, 1, 3])
def test_zerocopy_mode(batch):
    """O3: the kernel writes straight into mapped pinned host memory."""
    n, i = 6000, 13
    assert np.array_equal(run_e2e(n, i, 21, mode=P.PRNG_MODE_ZEROCOPY, batch=batch), oracle.stream(n, i, 21))


def test_zerocopy_needs_aligned_rows():
    with pytest.raises(P.PrngError) as e:
        run_e2e(1001, 3, mode=P.PRNG_MODE_ZEROCOPY)
    assert e.value.code == P.PRNG_EINVAL


@pytest.mark.parametrize("kind", [1, 2])
def test_host_memory_kinds(kind):
    """Write-combined and THP-registered pinned halves give the same stream."""
    n, i = 4096 + 8, 9
    count = n
    h = P.prng_create(n, 3)
    try:
        P.prng_set_option(h, P.PRNG_OPT_HOST_MEM, kind)
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 2)
        out = np.zeros((i, count), np.uint64)
        P.prng_init(h)
        P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), count, 0, i, 0))
    finally:
        P.prng_destroy(h)
    assert np.array_equal(out, oracle.stream(n, i, 3))


@pytest.mark.parametrize("kname", STAR_NAMES)
def test_star_output_all_paths(kname):
    """NEXT-3 (A19): scrambled output through e2e (O2, O3) and device-only, vs the oracle."""
    kv = _kid(kname)
    n, i = 4100, 7
    want = oracle.stream_star(n, i, 6)
    for mode in (P.PRNG_MODE_OVERLAP2, P.PRNG_MODE_ZEROCOPY):
        h = P.prng_create(n, 6)
        try:
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, kv)
            P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 1)
            P.prng_set_option(h, P.PRNG_OPT_MODE, mode)
            P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 3)
            out = np.zeros((i, n), np.uint64)
            P.prng_init(h)
            P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
            assert np.array_equal(out, want)
            # the state stays the plain recurrence
            assert np.array_equal(P.prng_read_state(h, n), oracle.stream(n, i, 6)[-1])
        finally:
            P.prng_destroy(h)
    h = P.prng_create(n, 6)
    try:
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, kv)
        P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 1)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, 8)
        P.prng_init(h)
        P.prng_generate(h, i)
        _, _, _, first, _ = P.prng_device_ring(h)
        for k in range(i):
            assert np.array_equal(P.prng_read_slot(h, (first + k) % 8, n), want[k])
    finally:
        P.prng_destroy(h)


def test_star_output_any_variant_any_order():
    """Every variant has the scrambled-output instantiation: OUTPUT = 1 is accepted before
    or after PRNG_OPT_KERNEL, and out-of-range values are still rejected."""
    h = P.prng_create(64, 0)
    try:
        for name in ALL_NAMES:
            P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 0)
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(name))
            P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 1)
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, 0)
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(name))
        with pytest.raises(P.PrngError):
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, len(ALL_NAMES))
    finally:
        P.prng_destroy(h)


# ---------------------------------------------------------------- NEXT-4: time-parallel jump-ahead
@pytest.mark.parametrize("n", [1, 33, 1000, 4099])
@pytest.mark.parametrize("i", [150, 300, 1001, 2600])
def test_time_parallel_device_only(n, i):
    """Small numrn: the launch is cut into iteration chunks started by GF(2) jump-ahead.
    Every output of every iteration vs the oracle, and the final state."""
    import torch
    pitch = (n + 3) // 4 * 4
    buf = torch.zeros((i, pitch), dtype=torch.int64, device="cuda")
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_init(h)
        P.prng_generate_device(h, i, buf.data_ptr(), pitch, i, 0)
        torch.cuda.synchronize()
        want = oracle.stream(n, i, SEED_PARITY)
        assert np.array_equal(buf[:, :n].cpu().numpy().view(np.uint64), want)
        assert np.array_equal(P.prng_read_state(h, n), want[-1])
    finally:
        P.prng_destroy(h)


@pytest.mark.parametrize("batch", [0, 700, 1])
@pytest.mark.parametrize("kname", ["auto", "v4n8s1a", "v2n4s1", "v2n32s1"])
def test_time_parallel_e2e_and_split(batch, kname):
    """Chunked batches (alternating e = 0 / 1 jump offsets), split calls, several variants."""
    n, i = 1000, 3000
    want = oracle.stream(n, i, 17)
    got = run_e2e(n, i, 17, batch=batch, kernel=_kid(kname), calls=[1000, 1313, 687])
    assert np.array_equal(got, want)


def test_time_parallel_off_is_identical():
    n, i = 777, 1400
    outs = []
    for tp in (0, 1):
        h = P.prng_create(n, 5)
        try:
            P.prng_set_option(h, P.PRNG_OPT_TIME_PARALLEL, tp)
            out = np.zeros((i, n), np.uint64)
            P.prng_init(h)
            P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
            outs.append(out)
        finally:
            P.prng_destroy(h)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], oracle.stream(n, i, 5))


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("chunk", [0, 1, 37, 300])
@pytest.mark.parametrize("kname", ["v4n4s1", "v4n8s1a", "v2n4s1"])
def test_forced_chunks_and_piece_order(kname, chunk, order):
    """PRNG_OPT_CHUNK_ITERS (jump-started chunks at any numrn) and PRNG_OPT_PIECE_ORDER
    (CTA-blocked dealing) change only the work order: every output, split calls included,
    and the final state vs the oracle; ragged numrn spanning several rounds of pieces."""
    n, i = 70001, 777
    want = oracle.stream(n, i, SEED_PARITY)
    for calls in ([i], [400, 1, 376]):
        h = P.prng_create(n, SEED_PARITY)
        try:
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(kname))
            P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, chunk)
            P.prng_set_option(h, P.PRNG_OPT_PIECE_ORDER, order)
            P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, 96)  # several rounds per warp
            out = np.zeros((i, n), np.uint64)
            sink = P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0)
            P.prng_init(h)
            for c in calls:
                P.prng_generate(h, c, P.SINK_COPY, sink)
            st = P.prng_read_state(h, n)
        finally:
            P.prng_destroy(h)
        assert np.array_equal(out, want), (calls, chunk, order)
        assert np.array_equal(st, want[-1])


@pytest.mark.parametrize("out_kind", [0, 1])
@pytest.mark.parametrize("epoch", [1, 3, 64])
@pytest.mark.parametrize("kname", STAR_NAMES)
def test_epoch_order(kname, epoch, out_kind):
    """PRNG_OPT_EPOCH_ITERS (epoch-major order: each warp runs its pieces E iterations at a
    time, the state through HBM between epochs): every
    output of every iteration, split calls, both output transforms, the final state; ragged
    numrn over several pieces per warp, and numrn with one piece per warp."""
    for n, warps in ((70001, 96), (5000, 64)):
        i = 777
        want = (oracle.stream_star if out_kind else oracle.stream)(n, i, SEED_PARITY)
        state = oracle.stream(n, i, SEED_PARITY)[-1]
        for calls in ([i], [400, 1, 376]):
            h = P.prng_create(n, SEED_PARITY)
            try:
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(kname))
                P.prng_set_option(h, P.PRNG_OPT_OUTPUT, out_kind)
                P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, epoch)
                P.prng_set_option(h, P.PRNG_OPT_TIME_PARALLEL, 0)
                P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, warps)
                out = np.zeros((i, n), np.uint64)
                sink = P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0)
                P.prng_init(h)
                for c in calls:
                    P.prng_generate(h, c, P.SINK_COPY, sink)
                st = P.prng_read_state(h, n)
            finally:
                P.prng_destroy(h)
            assert np.array_equal(out, want), (n, calls)
            assert np.array_equal(st, state)


# (numrn, iterations, ring slots, epoch option, expected (variant, epoch length)[, one-shot
# option]); L2 = 126 MB on B200; persistent grid 592 warps, one-shot grid 1776 resident warps:
# live set = R x min(resident warps, pieces) x bytes per warp-iteration vs 2 x L2.
ANTI_ABSORPTION = [
    (300007, 1000, 16, 0, ("v4n4s1p", 16)),  # no wide variant clears 2 x L2 and the widest has < 1 piece
                                             # per warp: epoch order on the default, E = R
    (300007, 1000, 16, -1, ("v4n4s1p", 0)),  # -1: natural order (absorbing) on request
    (300007, 40, 64, 0, ("v4n4s1p", 0)),     # no wrap inside the launch: nothing to absorb
    (1 << 20, 80, 64, 0, ("v2n32s1", 0)),    # 64 x 592 x 8 KiB = 310 MB: the 8 KiB variant
    (1 << 20, 310, 300, 0, ("v4n4s1p", 0)),  # one-shot grid (8192 pieces >= 4 waves): its resident set
                                             # 300 x 1776 x 1 KiB = 545 MB clears 2 x L2 unchanged
    (1 << 20, 310, 300, 0, ("v4n8s1", 0), 0),  # persistent grid: 300 x 592 x 2 KiB = 364 MB, the 2 KiB variant
    ((1 << 20) + 77, 80, 64, 0, ("v2n32s1", 0)),  # ragged
    (1 << 20, 50, 8, 0, ("v2n32s1", 8)),     # none clears 2 x L2: epoch order on the widest, E = R
    (1 << 21, 100, 40, 0, ("v2n32s1", 0)),   # widest at 8 warps/SM: 40 x 1184 x 8 KiB = 388 MB
]


def _slot_digest(row):
    """Per-iteration XOR and wrapping sum of one ring slot (numpy uint64 sums wrap)."""
    return int(np.bitwise_xor.reduce(row)), int(row.sum(dtype=np.uint64))


@pytest.mark.parametrize("case", ANTI_ABSORPTION)
@pytest.mark.parametrize("out_kind", [0, 1])
def test_anti_absorption_rule(case, out_kind):
    """The device-only launch wraps a ring of R slots: the default variant is replaced by a
    wider one (or epoch order) so that no address is rewritten while its line can still be
    in L2.  The kernel that ran (prng_last_launch), the R slots still in the
    ring (element by element for small runs, else per-slot XOR / sum digests against the
    oracle's per-iteration digests plus sampled elements) and the final state."""
    n, i, R, epoch_opt, expect = case[:5]
    one_shot = case[5] if len(case) > 5 else 1
    small = n * i <= 1 << 26
    if out_kind and not small:
        pytest.skip("scrambled output checked on the small cases")
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, one_shot)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, R)
        P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, epoch_opt)
        P.prng_set_option(h, P.PRNG_OPT_OUTPUT, out_kind)
        P.prng_init(h)
        P.prng_generate(h, i)
        ran, epoch = P.prng_last_launch(h)
        assert (P.prng_kernel_variant_name(ran), epoch) == expect
        _, _, _, first, _ = P.prng_device_ring(h)
        ks = range(max(0, i - R), i)
        rows = {k: P.prng_read_slot(h, (first + k) % R, n) for k in ks}
        st = P.prng_read_state(h, n)
    finally:
        P.prng_destroy(h)
    if small:
        want = (oracle.stream_star if out_kind else oracle.stream)(n, i, SEED_PARITY)
        for k in ks:
            assert np.array_equal(rows[k], want[k]), k
        assert np.array_equal(st, oracle.stream(n, i, SEED_PARITY)[-1])
    else:
        wx, ws = oracle.digest(n, i, SEED_PARITY)
        g = np.random.default_rng(3).integers(0, n, 200)
        for k in ks:
            assert _slot_digest(rows[k]) == (int(wx[k]), int(ws[k])), k
        for x in g:
            assert int(rows[i - 1][x]) == oracle.sample(int(x), i - 1, SEED_PARITY)
            assert int(st[x]) == oracle.sample(int(x), i - 1, SEED_PARITY)


@pytest.mark.parametrize("n,name", [(1 << 24, "v4n8s1a"), ((1 << 21) - 1, "v4n4s1p"), (1 << 21, "v4n8s1a"),
                                    ((1 << 21) + 300, "v4n8s1a"), (1 << 15, "v4n4s1p"), ((1 << 15) - 1, "v2n2s1")])
def test_auto_kernel_at_bench_shape(n, name):
    """"auto" (id 0): v4n8s1a from 2^21 work-items, v4n4s1p from 2^15, v2n2s1 below.  At the bench shape
    (2^24 x 1000, default 64 GiB ring = 512 slots) the live set is 512 x 592 x 2 KiB =
    620 MB > 2 x L2, so v4n8s1 runs in natural order; the last iteration and the state vs
    the oracle (sampled gids)."""
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_init(h)
        P.prng_generate(h, 1000)
        base, pitch, slots, first, end = P.prng_device_ring(h)
        ran, epoch = P.prng_last_launch(h)
        assert (P.prng_kernel_variant_name(ran), epoch) == (name, 0)
        if n == 1 << 24:
            assert slots == 512
            # 65536 pieces, 37 waves of one-shot warps (3 CTAs of 4 warps per SM) -> one piece per warp
            assert P.prng_last_grid(h) == (16384, 128, 1, True)
        import torch
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        pieces = -(-n // (32 * {"v4n8s1a": 8, "v4n4s1p": 4, "v2n2s1": 2}[name]))
        assert P.prng_last_grid(h)[3] == (pieces >= 4 * 3 * 4 * sms), (n, pieces)  # kOneShotMinWaves
        last = P.prng_read_slot(h, (first + 999) % slots, n)
        g = np.random.default_rng(5).integers(0, n, 2000)
        want = np.array([oracle.sample(int(x), 999, SEED_PARITY) for x in g], dtype=np.uint64)
        assert np.array_equal(last[g], want)
        assert np.array_equal(P.prng_read_state(h, n)[g], want)
    finally:
        P.prng_destroy(h)


def test_forced_chunks_device_only_bench_shape():
    """Forced chunks + CTA-blocked order at the bench width (2^24), device-only into a
    torch buffer: every iteration's XOR, wrapping sum and gid-weighted sum of all 2^24
    outputs (folded on the GPU) vs the oracle, and the final state element by element."""
    import torch
    n, i = 1 << 24, 48
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, 10)
        P.prng_set_option(h, P.PRNG_OPT_PIECE_ORDER, 1)
        buf = torch.empty((i, n), dtype=torch.int64, device="cuda")
        P.prng_init(h)
        P.prng_generate_device(h, i, buf.data_ptr(), n, i, 0)
        torch.cuda.synchronize()
        got = [_gpu_folds(buf[k], 0) for k in range(i)]
        last = buf[-1].cpu().numpy().view(np.uint64)
        st = P.prng_read_state(h, n)
    finally:
        P.prng_destroy(h)
    want = _oracle_folds_threads(n, i, SEED_PARITY, last=True)
    for k in range(i):
        assert got[k] == (int(want["xor"][k]), int(want["sum"][k]), int(want["wsum"][k])), k
    assert np.array_equal(last, want["last"]) and np.array_equal(st, want["last"])


@pytest.mark.parametrize("slots", [1, 7, 300])
@pytest.mark.parametrize("chunk", [0, 3])
def test_chunks_never_race_on_a_wrapping_ring(slots, chunk):
    """Time-parallel chunks of one piece run on different warps at once; on a ring with
    fewer slots than the launch's iterations two chunks would write the same slot, so the
    library keeps chunking to launches that do not wrap.  Small numrn (time-parallel by
    default from 144 iterations: >= 3 chunks of >= 48) and forced chunks through wrapping rings: the last R
    iterations and the state vs the oracle."""
    n, i = 100, 1000
    want = oracle.stream(n, i, 21)
    h = P.prng_create(n, 21)
    try:
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
        P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, chunk)
        P.prng_init(h)
        P.prng_generate(h, i)
        _, _, R, first, _ = P.prng_device_ring(h)
        for k in range(i - R, i):
            assert np.array_equal(P.prng_read_slot(h, (first + k) % R, n), want[k]), k
        assert np.array_equal(P.prng_read_state(h, n), want[-1])
    finally:
        P.prng_destroy(h)


@pytest.mark.parametrize("out_kind", [0, 1])
@pytest.mark.parametrize("kname", ["v4n8s1a", "v4n4s1p"])
def test_full_pieces_even_and_odd_iterations(kname, out_kind):
    """numrn a multiple of the piece size (every round uniform: the .aligned barrier of
    v4n8s1a, the two-iteration ping-pong loop of v4n4s1p).  Even and odd iteration counts,
    split calls (the first launch starts with the seeds, later ones with a step), end to
    end and device only, both output transforms, and a grid with several rounds per warp,
    vs the oracle."""
    for n in (1 << 16, 3 * 1024 * 37):   # multiples of 32 x 8 numbers
        i = 301
        want = (oracle.stream_star if out_kind else oracle.stream)(n, i, SEED_PARITY)
        state = oracle.stream(n, i, SEED_PARITY)[-1]
        for calls in ([i], [1, 2, 150, 148]):
            h = P.prng_create(n, SEED_PARITY)
            try:
                P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(kname))
                P.prng_set_option(h, P.PRNG_OPT_OUTPUT, out_kind)
                P.prng_set_option(h, P.PRNG_OPT_GRID_WARPS, 40)
                out = np.zeros((i, n), np.uint64)
                sink = P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0)
                P.prng_init(h)
                for c in calls:
                    P.prng_generate(h, c, P.SINK_COPY, sink)
                assert np.array_equal(out, want), (n, calls)
                assert np.array_equal(P.prng_read_state(h, n), state)
                P.prng_init(h)  # device only through the ring (no wrap: 301 < slots)
                for c in calls:
                    P.prng_generate(h, c)
                _, _, R, first, _ = P.prng_device_ring(h)
                for k in (0, 1, i // 2, i - 1):
                    assert np.array_equal(P.prng_read_slot(h, (first + k) % R, n), want[k]), k
                assert np.array_equal(P.prng_read_state(h, n), state)
            finally:
                P.prng_destroy(h)


@pytest.mark.parametrize("kname", STAR_NAMES)
def test_time_parallel_star(kname):
    kv = _kid(kname)
    n, i = 512, 1333
    h = P.prng_create(n, 2)
    try:
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, kv)
        P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 1)
        out = np.zeros((i, n), np.uint64)
        P.prng_init(h)
        P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
    finally:
        P.prng_destroy(h)
    assert np.array_equal(out, oracle.stream_star(n, i, 2))


@pytest.mark.parametrize("fused", [0, 1])
def test_nonblocking_accumulated_profile(fused):
    """bench.py's timed loop: PRNG_OPT_BLOCKING 0 + PRNG_OPT_PROFILE 2 -- K runs enqueued
    back to back, intervals accumulated, results identical; one launch per run when a1 is
    fused, two (seed + batch) when not."""
    import torch
    n, i, K = 5000, 40, 3
    h = P.prng_create(n, 8)
    try:
        P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, fused)
        P.prng_set_option(h, P.PRNG_OPT_PROFILE, 2)
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 0)
        for _ in range(K):
            P.prng_init(h)
            P.prng_generate(h, i)
        torch.cuda.synchronize()
        ids, s, e, _ = P.prng_prof_events(h)
        assert (ids == 0).sum() == K * (1 - fused) and (ids == 1).sum() == K and (e >= s).all()
        P.prng_set_option(h, P.PRNG_OPT_BLOCKING, 1)
        assert np.array_equal(P.prng_read_state(h, n), oracle.stream(n, i, 8)[-1])
    finally:
        P.prng_destroy(h)


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (read-only use)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": "<i8", "version": 3}


# ---------------------------------------------------------------- shared host output (north_star e)
def test_generate_host_shards_fill_one_array():
    """Each 'rank' (one handle per gid shard) writes its columns of one host array directly."""
    n, i, world = 10007, 9, 3
    arr = np.zeros((i, n), np.uint64)
    for r in range(world):
        b, c = shard_range(n, r, world)
        h = P.prng_create_range(n, SEED_PARITY, b, c)
        try:
            P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 2)
            P.prng_init(h)
            P.prng_generate_host(h, i, arr, n, i, col_offset=b)
        finally:
            P.prng_destroy(h)
    assert np.array_equal(arr, oracle.stream(n, i, SEED_PARITY))


def test_generate_host_row_ring_and_continuation():
    """dst_rows < numiter wraps; a second call continues the stream into its own rows."""
    n, i, rows = 3000, 11, 4
    want = oracle.stream(n, 2 * i, 4)
    arr = np.zeros((rows, n), np.uint64)
    h = P.prng_create(n, 4)
    try:
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 3)
        P.prng_init(h)
        P.prng_generate_host(h, i, arr, n, rows)
        for k in range(i - rows, i):
            assert np.array_equal(arr[k % rows], want[k])
        P.prng_generate_host(h, i, arr, n, rows)
        for k in range(i - rows, i):
            assert np.array_equal(arr[k % rows], want[i + k])
    finally:
        P.prng_destroy(h)


def _rank_writes_shm(rank, world, n, i, shm_name):
    import numpy as _np
    from multiprocessing import shared_memory
    import paper_1609_01257_b200 as _P
    from workloads import shard_range as _sr
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        arr = _np.ndarray((i, n), dtype=_np.uint64, buffer=shm.buf)
        b, c = _sr(n, rank, world)
        h = _P.prng_create_range(n, 7, b, c, 0)
        try:
            _P.prng_init(h)
            _P.prng_generate_host(h, i, arr, n, i, col_offset=b)
        finally:
            _P.prng_destroy(h)
        del arr
    finally:
        shm.close()


def test_two_processes_write_one_shared_host_array():
    """Two processes (ranks) on cuda:0, one POSIX shared-memory output array: each D2H's its
    gid columns straight into it; the parent sees the single-device stream."""
    import multiprocessing as mp
    from multiprocessing import shared_memory
    n, i, world = 4099, 6, 2
    shm = shared_memory.SharedMemory(create=True, size=8 * n * i)
    try:
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=_rank_writes_shm, args=(r, world, n, i, shm.name)) for r in range(world)]
        [p.start() for p in ps]
        [p.join(timeout=300) for p in ps]
        assert all(p.exitcode == 0 for p in ps)
        arr = np.ndarray((i, n), dtype=np.uint64, buffer=shm.buf).copy()
        assert np.array_equal(arr, oracle.stream(n, i, 7))
    finally:
        shm.close()
        shm.unlink()


def test_python_sink_exception_propagates():
    """A Python sink that raises aborts generation (PRNG_ESINK inside) and the exception
    reaches the caller; the handle is poisoned until prng_init."""
    h = P.prng_create(100, 0)
    try:
        P.prng_init(h)

        def bad(*a):
            raise KeyError("consumer failed")
        with pytest.raises(KeyError):
            P.prng_generate(h, 5, bad)
        with pytest.raises(P.PrngError) as e:
            P.prng_generate(h, 1, P.SINK_NULL)
        assert e.value.code == P.PRNG_ESTATE
    finally:
        P.prng_destroy(h)


# ---------------------------------------------------------------- checkpoint / resume (prng_seek)
@pytest.mark.parametrize("k", [0, 1, 2, 7, 1000, 65537])
def test_seek_resumes_the_stream(k):
    n, m = 333, 600
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_seek(h, k)
        out = np.zeros((m, n), np.uint64)
        P.prng_generate(h, m, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, k, m, 0))
    finally:
        P.prng_destroy(h)
    assert np.array_equal(out, oracle.stream(n, k + m, SEED_PARITY)[k:])


def _xs_pow_columns(k):
    """Columns of T^k for the ORACLE's xs by binary exponentiation over GF(2) (test-side)."""
    cols = [oracle.xorshift64(1 << j) for j in range(64)]

    def apply(M, x):
        y = 0
        for j in range(64):
            if (x >> j) & 1:
                y ^= M[j]
        return y

    R = [1 << j for j in range(64)]
    B = cols
    while k:
        if k & 1:
            R = [apply(B, c) for c in R]
        B = [apply(B, c) for c in B]
        k >>= 1
    return R, apply


def test_seek_far_ahead():
    """k = 2^40 + 5: no oracle can step there; the expected state is xs^(k-1)(seed64) by a
    test-side GF(2) power of the oracle's own xs, then the stream continues by the oracle."""
    k = (1 << 40) + 5
    n, m = 64, 3
    R, apply = _xs_pow_columns(k - 1)
    h = P.prng_create(n, 1)
    try:
        P.prng_seek(h, k)
        st = P.prng_read_state(h, n)
        out = np.zeros((m, n), np.uint64)
        P.prng_generate(h, m, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, k, m, 0))
    finally:
        P.prng_destroy(h)
    for g in range(n):
        want = apply(R, oracle.seed64(g, 1))
        assert int(st[g]) == want
        x = want
        for t in range(m):
            x = oracle.xorshift64(x)
            assert int(out[t, g]) == x


def test_argument_errors_on_a_live_handle():
    """EINVAL paths that need a handle: option values, device-buffer layout, host array."""
    import torch
    h = P.prng_create(1000, 0)
    try:
        for opt, bad in [(P.PRNG_OPT_MODE, 9), (P.PRNG_OPT_KERNEL, 999), (P.PRNG_OPT_OUTPUT, 2),
                         (P.PRNG_OPT_RING_PAD, 3), (P.PRNG_OPT_HOST_MEM, 7), (P.PRNG_OPT_PROFILE, 5),
                         (P.PRNG_OPT_CTA_WARPS, 9), (P.PRNG_OPT_CHUNK_ITERS, -1), (P.PRNG_OPT_PIECE_ORDER, 2),
                         (P.PRNG_OPT_EPOCH_ITERS, -2), (99, 0)]:
            with pytest.raises(P.PrngError) as e:
                P.prng_set_option(h, opt, bad)
            assert e.value.code == P.PRNG_EINVAL, (opt, bad)
        for opt, good in [(P.PRNG_OPT_CHUNK_ITERS, 17), (P.PRNG_OPT_PIECE_ORDER, 1), (P.PRNG_OPT_EPOCH_ITERS, -1)]:
            P.prng_set_option(h, opt, good)
            assert P.prng_get_option(h, opt) == good
            P.prng_set_option(h, opt, 0)
        assert P.prng_last_launch(h) == (-1, 0)  # nothing launched yet
        P.prng_init(h)
        buf = torch.zeros(8 * 1024 + 8, dtype=torch.int64, device="cuda")
        for ptr, pitch in [(buf.data_ptr() + 8, 1000), (buf.data_ptr(), 1001), (buf.data_ptr(), 996)]:
            with pytest.raises(P.PrngError) as e:
                P.prng_generate_device(h, 2, ptr, pitch, 2)
            assert e.value.code == P.PRNG_EINVAL
        arr = np.zeros((2, 1000), np.uint64)
        with pytest.raises(P.PrngError):
            P.prng_generate_host(h, 0, arr, 1000, 2)
        with pytest.raises(P.PrngError):
            P.prng_generate_host(h, 2, arr, 999, 2)
        P.prng_generate_host(h, 2, arr, 1000, 2)    # still usable after rejected calls
        assert np.array_equal(arr, oracle.stream(1000, 2, 0))
    finally:
        P.prng_destroy(h)


def test_randomised_configurations():
    """Seeded fuzz over the option space: numrn, numiter, seed, mode, batch size, kernel
    variant, output transform, time-parallel on/off, epoch order (auto / off / forced E),
    piece order, jump-started chunks, fused or separate a1, and how the run is split into
    calls; end to end
    (every output) or device only (the ring slots still held, small rings that wrap);
    every value vs the oracle."""
    r = np.random.default_rng(20261017)
    nvar = P.prng_kernel_variants()
    names = [P.prng_kernel_variant_name(k) for k in range(nvar)]
    usable = list(range(nvar))
    for trial in range(60):
        n = int(r.choice([1, 2, 3, 31, 64, 100, 1000, 4096, 5003, 20000, 70001]))
        i = int(r.choice([1, 2, 5, 17, 130, 600]))
        seed = int(r.integers(0, 1 << 63))
        mode = int(r.integers(0, 5))
        if mode == P.PRNG_MODE_ZEROCOPY and n % 4:
            mode = P.PRNG_MODE_OVERLAP2
        kv = int(r.choice(usable))
        star = int(r.random() < 0.3)
        tp = int(r.random() < 0.8)
        batch = int(r.choice([0, 1, 3, 50]))
        epoch = int(r.choice([0, 0, -1, 1, 7, 64]))
        order = int(r.random() < 0.3)
        chunk = int(r.choice([0, 0, 0, 3, 40]))
        device_only = bool(r.random() < 0.4)
        slots = int(r.choice([1, 2, 5, 16, 1000]))
        cuts = sorted({int(c) for c in r.integers(1, i, size=2)}) if i > 2 else []
        calls = [b - a for a, b in zip([0] + cuts, cuts + [i])]
        fused = int(r.random() < 0.7)
        cfg = dict(trial=trial, n=n, i=i, mode=mode, kernel=names[kv], star=star, tp=tp, batch=batch, epoch=epoch,
                   order=order, chunk=chunk, device_only=device_only, slots=slots, calls=calls, fused=fused)
        want = oracle.stream_star(n, i, seed) if star else oracle.stream(n, i, seed)
        h = P.prng_create(n, seed)
        try:
            for opt, val in [(P.PRNG_OPT_MODE, mode), (P.PRNG_OPT_KERNEL, kv), (P.PRNG_OPT_OUTPUT, star),
                             (P.PRNG_OPT_TIME_PARALLEL, tp), (P.PRNG_OPT_BATCH_ITERS, batch),
                             (P.PRNG_OPT_EPOCH_ITERS, epoch), (P.PRNG_OPT_PIECE_ORDER, order),
                             (P.PRNG_OPT_CHUNK_ITERS, chunk), (P.PRNG_OPT_FUSED_SEED, fused)]:
                P.prng_set_option(h, opt, val)
            if device_only:
                P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
                P.prng_init(h)
                for c in calls:
                    P.prng_generate(h, c)
                _, _, R, first, end = P.prng_device_ring(h)
                assert end == i, cfg
                for k in range(max(0, i - R), i):
                    assert np.array_equal(P.prng_read_slot(h, (first + k) % R, n), want[k]), (cfg, k)
            else:
                out = np.zeros((i, n), np.uint64)
                sink = P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0)
                P.prng_init(h)
                for c in calls:
                    P.prng_generate(h, c, P.SINK_COPY, sink)
                assert np.array_equal(out, want), cfg
            assert np.array_equal(P.prng_read_state(h, n), oracle.stream(n, i, seed)[-1]), cfg
        finally:
            P.prng_destroy(h)



# ---------------------------------------------------------------- full shapes, order-sensitive
M64 = (1 << 64) - 1


def _oracle_folds_threads(n, i, seed, gid_begin=0, count=None, last=False, nthreads=None, shard=1 << 26):
    """oracle.folds on contiguous gid shards of [gid_begin, gid_begin + count) (at most
    `shard` gids each, so host memory stays bounded) over a pool of threads (ctypes releases
    the GIL).  The folds combine across shards: XOR, wrapping sum, and the gid-weighted sum
    (its weights use the global gid); `last` concatenates."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    count = n - gid_begin if count is None else count
    nthreads = nthreads or max(1, len(os.sched_getaffinity(0)))
    nshards = max(nthreads, (count + shard - 1) // shard)
    spans = [shard_range(count, r, nshards) for r in range(nshards)]

    def work(span):
        b, c = span
        return oracle.folds(n, i, seed, gid_begin=gid_begin + b, count=c, last=last) if c else None

    with ThreadPoolExecutor(nthreads) as ex:
        res = list(ex.map(work, spans))
    out = {"xor": np.zeros(i, np.uint64), "sum": np.zeros(i, np.uint64), "wsum": np.zeros(i, np.uint64)}
    for rr in res:
        if rr is not None:
            out["xor"] ^= rr["xor"]
            out["sum"] += rr["sum"]
            out["wsum"] += rr["wsum"]
    if last:
        out["last"] = np.concatenate([rr["last"] for rr in res if rr is not None])
    return out


def _gpu_folds(row, gid0, chunk=1 << 27):
    """(xor, sum, gid-weighted sum) of one int64 CUDA row whose element j is gid gid0 + j,
    folded chunk by chunk (bounded temporaries); torch's int64 arithmetic wraps mod 2^64
    (two's complement), which is the oracle's u64 arithmetic."""
    import torch
    x = s = w = 0
    for c0 in range(0, row.numel(), chunk):
        part = row[c0:c0 + chunk]
        wt = torch.arange(part.numel(), dtype=torch.int64, device=part.device) * 2 + (2 * (gid0 + c0) + 1)
        s += int(part.sum().item())
        w += int((part * wt).sum().item())
        del wt
        v = part.clone()
        m = v.numel()
        while m > 1:
            h2 = m // 2
            v[:h2] ^= v[m - h2:m]
            m -= h2
        x ^= int(v[0].item()) & M64
        del v
    return x & M64, s & M64, w & M64


def _device_only_full_shape(numrn_total, gid_begin, count, numiter, seed, expect_kernel=None, one_shot=1,
                            expect_one_shot=None):
    """One device-only launch exactly as bench.py runs it (default kernel, default 64 GiB
    rotating ring; PRNG_OPT_ONE_SHOT as given): for every iteration still in the ring, the
    XOR, the wrapping sum and the gid-weighted sum of all its outputs (order-sensitive: a
    misplaced piece changes it), and the whole last iteration and the final state element by
    element -- all against the oracle's flat loop over the same gid range."""
    import torch
    h = P.prng_create_range(numrn_total, seed, gid_begin, count, 0)
    try:
        P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, one_shot)
        P.prng_init(h)
        P.prng_generate(h, numiter)
        ran, epoch = P.prng_last_launch(h)
        if expect_kernel is not None:
            assert (P.prng_kernel_variant_name(ran), epoch) == expect_kernel
        if expect_one_shot is not None:
            blocks, threads, rounds, os_ = P.prng_last_grid(h)
            assert os_ == expect_one_shot and (rounds == 1 if os_ else blocks <= 148 * 8), (blocks, threads, rounds)
        base, pitch, slots, first, end = P.prng_device_ring(h)
        assert end == numiter
        ring = torch.as_tensor(_DevArray(base, (slots, pitch)), device="cuda")
        got = {k: _gpu_folds(ring[(first + k) % slots, :count], gid_begin) for k in range(max(0, numiter - slots), numiter)}
        last = ring[(first + numiter - 1) % slots, :count].cpu().numpy().view(np.uint64).copy()
        st = P.prng_read_state(h)
        del ring
    finally:
        P.prng_destroy(h)
    want = _oracle_folds_threads(numrn_total, numiter, seed, gid_begin, count, last=True)
    for k, (x, s, ws) in got.items():
        assert (x, s, ws) == (int(want["xor"][k]), int(want["sum"][k]), int(want["wsum"][k])), k
    assert np.array_equal(last, want["last"]), "last iteration differs from the oracle"
    assert np.array_equal(st, want["last"]), "final state differs from the oracle"
    # and, by an independent route (the random-access form xs^k(seed64(g))), sampled gids
    g, k = sample_points(numrn_total, numiter, 200, rng_seed=99, gid_begin=gid_begin, count=count)
    for gg in g[:200]:
        assert int(st[gg - gid_begin]) == oracle.sample(int(gg), numiter - 1, seed)


@pytest.mark.slow
@pytest.mark.parametrize("one_shot", [1, 0])
def test_config2_bench_shape_order_sensitive(one_shot):
    """BASELINE config 2 = the bench step (numrn = 2^24, numiter = 1000, seed 0, the default
    kernel "auto" -> v4n8s1a, 512-slot ring; by default on a one-shot grid, and on the
    persistent grid with PRNG_OPT_ONE_SHOT 0): every ring slot's three folds, the whole last
    iteration and the state element by element, vs the oracle."""
    _device_only_full_shape(1 << 24, 0, 1 << 24, 1000, 0, ("v4n8s1a", 0), one_shot, bool(one_shot))


@pytest.mark.slow
@pytest.mark.parametrize("lg,name,one_shot", [(25, "v4n8s1a", 1), (26, "v4n8s1a", 1), (27, "v4n16s1", 1),
                                              (25, "v4n8s1a", 0), (26, "v4n16s1", 0), (27, "v2n32s1", 0)])
def test_config4_rank_shapes_order_sensitive(lg, name, one_shot):
    """BASELINE config 4 at its per-rank shapes: 2^28 over P = 8 / 4 / 2 ranks gives 2^25 /
    2^26 / 2^27 gids per rank, 1000 iterations, default 64 GiB ring of 256 / 128 / 64 slots.
    By default a one-shot grid (1776 resident warps), on v4n8s1a while its live set clears
    2 x L2 and on v4n16s1 at 64 slots (64 x 1776 x 2 KiB = 233 MB would not); on the
    persistent grid (PRNG_OPT_ONE_SHOT 0, 592 warps) the anti-absorption rule picks
    v4n8s1a / v4n16s1 / v2n32s1.  The LAST rank's gid range (up to gid 2^28 - 1), so the global-gid
    weights and the gid offset are exercised."""
    n = 1 << lg
    P_ = (1 << 28) // n
    b, c = shard_range(1 << 28, P_ - 1, P_)
    _device_only_full_shape(1 << 28, b, c, 1000, SEED_PARITY, (name, 0), one_shot, bool(one_shot))


def _e2e_digest_run(numrn_total, gid_begin, count, numiter, seed, mode):
    """End to end through prng_generate with the digest sink (xor / sum / gid-weighted sum
    per iteration, folded on the host from the pinned batches) and the final state."""
    xo, so, wo = (np.zeros(numiter, np.uint64) for _ in range(3))
    d = P.DigestSink(xo.ctypes.data_as(P.P64), so.ctypes.data_as(P.P64), 0, numiter, wo.ctypes.data_as(P.P64))
    h = P.prng_create_range(numrn_total, seed, gid_begin, count, 0)
    try:
        P.prng_set_option(h, P.PRNG_OPT_MODE, mode)
        P.prng_init(h)
        P.prng_generate(h, numiter, P.SINK_DIGEST, d)
        st = P.prng_read_state(h)
    finally:
        P.prng_destroy(h)
    return xo, so, wo, st


@pytest.mark.slow
def test_config3_full_e2e_order_sensitive():
    """BASELINE config 3 in full: 2^24 x 1000 end to end through the default O2 pipeline
    (134 GB over the host link); every iteration's three folds and the final state vs the
    oracle."""
    n, i = 1 << 24, 1000
    xo, so, wo, st = _e2e_digest_run(n, 0, n, i, SEED_PARITY, P.PRNG_MODE_OVERLAP2)
    want = _oracle_folds_threads(n, i, SEED_PARITY, last=True)
    assert np.array_equal(xo, want["xor"]) and np.array_equal(so, want["sum"]) and np.array_equal(wo, want["wsum"])
    assert np.array_equal(st, want["last"])


@pytest.mark.slow
@pytest.mark.parametrize("mode", [P.PRNG_MODE_OVERLAP2, P.PRNG_MODE_ZEROCOPY])
def test_config5_rank_shape_e2e_order_sensitive(mode):
    """BASELINE config 5 at its per-rank shape: rank 3 of 8 of the 2^28 stream (2^25 gids
    from gid 3 x 2^25), 100 iterations, end to end through the pinned double buffer (O2) and
    through zero-copy (O3): every iteration's three folds and the final state vs the oracle
    over the same gid range (the paper's read / out pipeline)."""
    n, i = 1 << 28, 100
    b, c = shard_range(n, 3, 8)
    xo, so, wo, st = _e2e_digest_run(n, b, c, i, SEED_PARITY, mode)
    want = _oracle_folds_threads(n, i, SEED_PARITY, b, c, last=True)
    assert np.array_equal(xo, want["xor"]) and np.array_equal(so, want["sum"]) and np.array_equal(wo, want["wsum"])
    assert np.array_equal(st, want["last"])


@pytest.mark.slow
def test_config2_every_iteration_no_ring():
    """The bench kernel at the bench shape (2^24 x 1000, one launch, default variant and
    grid) into a 134 GB device buffer with one slot per iteration (no wrap): all 1000
    iterations folded on the GPU (XOR, wrapping sum, gid-weighted sum) vs the oracle."""
    import torch
    n, i = 1 << 24, 1000
    free, _ = torch.cuda.mem_get_info()
    if free < 8 * n * i + (4 << 30):
        pytest.skip("needs ~140 GB of free device memory")
    buf = torch.empty((i, n), dtype=torch.int64, device="cuda")
    h = P.prng_create(n, 0)
    try:
        P.prng_init(h)
        P.prng_generate_device(h, i, buf.data_ptr(), n, i, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got = [_gpu_folds(buf[k], 0) for k in range(i)]
    finally:
        P.prng_destroy(h)
    del buf
    torch.cuda.empty_cache()
    want = _oracle_folds_threads(n, i, 0)
    for k in range(i):
        assert got[k] == (int(want["xor"][k]), int(want["sum"][k]), int(want["wsum"][k])), k


# ---------------------------------------------------------------- A3: the zero-state fix-up on the GPU
A3_GID, A3_SEED = 2654435716, 0x236D2904C6FC2D12   # derived in tests/test_oracle_pins.py::_a3_trigger


@pytest.mark.parametrize("case", ["e2e_default", "v2n4s1", "epoch", "time_parallel", "star", "zerocopy",
                                  "device_only"])
def test_a3_zero_fixup_on_gpu(case):
    """The seed kernel's 0 -> 1 fix-up (reading A3; PAPER.md P:173 needs
    nonzero seeds) at the one gid where the raw composition is 0: 2000 gids around it of the
    2^32 stream, element by element vs the oracle, through the default path, the 16-byte
    variant, epoch order, time-parallel chunks, the scrambled output, zero-copy and the
    device-only ring."""
    n, b, c = 1 << 32, A3_GID - 1000, 2000
    i = 600 if case == "time_parallel" else 9
    star = case == "star"
    want = (oracle.stream_star if star else oracle.stream)(n, i, A3_SEED, gid_begin=b, count=c)
    plain = oracle.stream(n, i, A3_SEED, gid_begin=b, count=c)
    assert plain[0, 1000] == 1 and plain[1, 1000] == 1082269761
    h = P.prng_create_range(n, A3_SEED, b, c, 0)
    try:
        if case == "v2n4s1":
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid("v2n4s1"))
        if case == "star":
            P.prng_set_option(h, P.PRNG_OPT_OUTPUT, 1)
        if case == "zerocopy":
            P.prng_set_option(h, P.PRNG_OPT_MODE, P.PRNG_MODE_ZEROCOPY)
        if case in ("epoch", "device_only"):
            P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, i)
            if case == "epoch":
                P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, 3)
                P.prng_set_option(h, P.PRNG_OPT_TIME_PARALLEL, 0)
            P.prng_init(h)
            P.prng_generate(h, i)
            ran, epoch = P.prng_last_launch(h)
            assert epoch == (3 if case == "epoch" else 0)
            _, _, R, first, _ = P.prng_device_ring(h)
            out = np.stack([P.prng_read_slot(h, (first + k) % R) for k in range(i)])
        else:
            out = np.zeros((i, c), np.uint64)
            P.prng_init(h)
            P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), c, 0, i, b))
        st = P.prng_read_state(h)
    finally:
        P.prng_destroy(h)
    assert np.array_equal(out, want)
    assert np.array_equal(st, plain[-1])
    if not star:
        assert out[0, 1000] == 1


# ---------------------------------------------------------------- ABI robustness
def test_set_streams_validates_before_touching_the_handle():
    """prng_set_streams(NULL, NULL) / identical streams: PRNG_EINVAL and the handle keeps its
    own two streams -- generation afterwards still overlaps and is bit-exact."""
    import torch
    n, i = 5000, 12
    h = P.prng_create(n, 4)
    try:
        s = torch.cuda.Stream()
        for g, c in [(0, 0), (s.cuda_stream, 0), (0, s.cuda_stream), (s.cuda_stream, s.cuda_stream)]:
            with pytest.raises(P.PrngError) as e:
                P.prng_set_streams(h, g, c)
            assert e.value.code == P.PRNG_EINVAL
        out = np.zeros((i, n), np.uint64)
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 2)
        P.prng_init(h)
        P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
        assert np.array_equal(out, oracle.stream(n, i, 4))
        # valid torch streams are then accepted and used
        g2, c2 = torch.cuda.Stream(), torch.cuda.Stream()
        P.prng_set_streams(h, g2.cuda_stream, c2.cuda_stream)
        P.prng_init(h)
        P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, i, 0))
        assert np.array_equal(out, oracle.stream(n, i, 4))
    finally:
        P.prng_destroy(h)


@pytest.mark.parametrize("fail_at", [1, 2, 3, 4, 5, 9])
def test_generate_host_failure_poisons_the_handle(fail_at, monkeypatch):
    """A CUDA call of prng_generate_host that fails (fault injected at the fail_at-th checked
    call: stream waits, event records, the 2-D copies, event syncs) makes the call return
    PRNG_ECUDA and poisons the handle (PRNG_ESTATE) instead of returning silently; after
    prng_init the handle is bit-exact again."""
    monkeypatch.setenv("PRNG_B200_FAULT_AFTER", str(fail_at))
    n, i = 3000, 12
    h = P.prng_create(n, 6)
    try:
        P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 2)
        arr = np.zeros((i, n), np.uint64)
        P.prng_init(h)
        with pytest.raises(P.PrngError) as e:
            P.prng_generate_host(h, i, arr, n, i)
        assert e.value.code == P.PRNG_ECUDA
        with pytest.raises(P.PrngError) as e:
            P.prng_generate_host(h, i, arr, n, i)
        assert e.value.code == P.PRNG_ESTATE
        P.prng_init(h)
        P.prng_generate_host(h, i, arr, n, i)   # the injected fault fired once
        assert np.array_equal(arr, oracle.stream(n, i, 6))
    finally:
        P.prng_destroy(h)


def test_binding_checks_host_buffer_sizes():
    """The Python binding refuses host arrays smaller than what the C side would write."""
    n = 1000
    h = P.prng_create(n, 0)
    try:
        P.prng_init(h)
        with pytest.raises(ValueError):
            P.prng_generate_host(h, 4, np.zeros((3, n), np.uint64), n, 4)       # 3 rows < 4
        with pytest.raises(ValueError):
            P.prng_generate_host(h, 2, np.zeros((2, n), np.uint64), n, 2, col_offset=1)
        with pytest.raises(ValueError):
            P.prng_read_state(h, n + 1)
        assert P.prng_get_range(h) == (n, 0, n)
        arr = np.zeros((2, n), np.uint64)
        P.prng_generate_host(h, 2, arr, n, 2)
        assert np.array_equal(arr, oracle.stream(n, 2, 0))
    finally:
        P.prng_destroy(h)


@pytest.mark.slow
def test_maximum_numrn_full_range():
    """The maximum size (A12: numrn = 2^32, every gid of the cl_uint range): one
    handle over all 2^32 work-items, 3 iterations device-only (a 3-slot ring of 32 GiB slots),
    every slot's XOR / sum / gid-weighted sum folded on the GPU vs the oracle (all 2^32 gids,
    sharded so host memory stays bounded), plus sampled gids (the top gid included) and the
    A3 gid vs the random-access form."""
    import torch
    n, i = 1 << 32, 3
    free, _ = torch.cuda.mem_get_info()
    if free < (4 * 8 << 32) + (8 << 30):
        pytest.skip("needs ~136 GB of free device memory")
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, i)
        P.prng_init(h)
        P.prng_generate(h, i)
        base, pitch, slots, first, end = P.prng_device_ring(h)
        assert (slots, end) == (i, i)
        ring = torch.as_tensor(_DevArray(base, (slots, pitch)), device="cuda")
        got = [_gpu_folds(ring[(first + k) % slots, :n], 0) for k in range(i)]
        g = [0, 1, A3_GID, n - 2, n - 1] + [int(x) for x in np.random.default_rng(4).integers(0, n, 200)]
        idx = torch.tensor(g, dtype=torch.int64, device="cuda")
        rows = [ring[(first + k) % slots].index_select(0, idx).cpu().numpy().view(np.uint64) for k in range(i)]
        del ring
    finally:
        P.prng_destroy(h)
    for k in range(i):
        for j, gg in enumerate(g):
            assert int(rows[k][j]) == oracle.sample(gg, k, SEED_PARITY), (k, gg)
    want = _oracle_folds_threads(n, i, SEED_PARITY)
    for k in range(i):
        assert got[k] == (int(want["xor"][k]), int(want["sum"][k]), int(want["wsum"][k])), k


def test_order_sensitive_fold_catches_a_misplaced_piece():
    """Why the full-shape tests fold with sum (2g + 1) x: swap two
    warp pieces (2 KiB each) of a correct GPU slot -- the XOR and the wrapping sum still
    match the oracle, the gid-weighted sum does not; a single flipped bit also fails it."""
    import torch
    n, i = 1 << 20, 4
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, i)
        P.prng_init(h)
        P.prng_generate(h, i)
        base, pitch, slots, first, _ = P.prng_device_ring(h)
        ring = torch.as_tensor(_DevArray(base, (slots, pitch)), device="cuda")
        row = ring[(first + i - 1) % slots, :n].clone()
    finally:
        P.prng_destroy(h)
    want = _oracle_folds_threads(n, i, SEED_PARITY)
    ok = (int(want["xor"][-1]), int(want["sum"][-1]), int(want["wsum"][-1]))
    assert _gpu_folds(row, 0) == ok
    bad = row.clone()
    bad[1000 * 256:1001 * 256], bad[3000 * 256:3001 * 256] = row[3000 * 256:3001 * 256], row[1000 * 256:1001 * 256]
    x, s, w = _gpu_folds(bad, 0)
    assert (x, s) == ok[:2] and w != ok[2]
    bad = row.clone()
    bad[12345] ^= 1 << 40
    assert _gpu_folds(bad, 0)[2] != ok[2]


def test_randomised_api_sequences():
    """Seeded fuzz over sequences of C-ABI calls on one handle: prng_init / prng_seek, then a
    random mix of prng_generate (sink or device-only ring), prng_generate_device (into a
    torch buffer, random pitch and slot count) and prng_generate_host (random row ring),
    with random variant / output / time-parallel / fused-seed options (and, sometimes, a
    state read between prng_init and the first generate); after every call the emitted
    iterations (and the state) are compared with the oracle's stream at those positions."""
    import torch
    r = np.random.default_rng(777)
    names = [P.prng_kernel_variant_name(k) for k in range(P.prng_kernel_variants())]
    for trial in range(40):
        n = int(r.choice([1, 5, 64, 129, 1000, 4099, 30001]))
        seed = int(r.integers(0, 1 << 63))
        star = int(r.random() < 0.3)
        start = int(r.choice([0, 0, 1, 7, 300]))
        total = start + 700
        want = (oracle.stream_star if star else oracle.stream)(n, total, seed)
        plain = oracle.stream(n, total, seed)
        h = P.prng_create(n, seed)
        try:
            P.prng_set_option(h, P.PRNG_OPT_KERNEL, int(r.integers(0, len(names))))
            P.prng_set_option(h, P.PRNG_OPT_OUTPUT, star)
            P.prng_set_option(h, P.PRNG_OPT_TIME_PARALLEL, int(r.random() < 0.8))
            P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, int(r.choice([0, 1, 3, 64])))
            P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, int(r.random() < 0.7))
            if start:
                P.prng_seek(h, start)
            else:
                P.prng_init(h)
                if r.random() < 0.3:  # the pending seeds, materialised by the read
                    assert np.array_equal(P.prng_read_state(h), plain[0]), trial
            pos = start
            while pos < total:
                m = int(min(total - pos, r.choice([1, 2, 9, 130, 300])))
                kind = int(r.integers(0, 4))
                ctx = dict(trial=trial, n=n, pos=pos, m=m, kind=kind, star=star)
                if kind == 0:    # end to end through the copy sink
                    out = np.zeros((m, n), np.uint64)
                    P.prng_generate(h, m, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, pos, m, 0))
                    assert np.array_equal(out, want[pos:pos + m]), ctx
                elif kind == 1:  # device only through the handle's ring
                    slots = int(r.choice([1, 3, 1000]))
                    P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
                    P.prng_generate(h, m)
                    _, _, R, first, end = P.prng_device_ring(h)
                    assert end == pos + m, ctx
                    for k in range(max(pos, pos + m - R), pos + m):
                        assert np.array_equal(P.prng_read_slot(h, (first + k) % R), want[k]), (ctx, k)
                elif kind == 2:  # device only into a caller-owned torch buffer
                    pitch = (n + 3) // 4 * 4 + 4 * int(r.integers(0, 3))
                    dslots = int(r.choice([m, max(1, m // 2), 1]))
                    buf = torch.zeros((dslots, pitch), dtype=torch.int64, device="cuda")
                    P.prng_generate_device(h, m, buf.data_ptr(), pitch, dslots, 0)
                    torch.cuda.synchronize()
                    got = buf[:, :n].cpu().numpy().view(np.uint64)
                    for t in range(max(0, m - dslots), m):
                        assert np.array_equal(got[t % dslots], want[pos + t]), (ctx, t)
                else:            # end to end straight into a host array (row ring)
                    rows = int(r.choice([m, 2, 1]))
                    arr = np.zeros((rows, n), np.uint64)
                    P.prng_generate_host(h, m, arr, n, rows)
                    for t in range(max(0, m - rows), m):
                        assert np.array_equal(arr[t % rows], want[pos + t]), (ctx, t)
                pos += m
                assert np.array_equal(P.prng_read_state(h), plain[pos - 1]), ctx
        finally:
            P.prng_destroy(h)


# ---------------------------------------------------------------- a1 fused into the batch launch
# PRNG_OPT_FUSED_SEED 1 (default): prng_init enqueues nothing and the next batch kernel
# computes seed64 in registers (prng_kernels.cuh start_states); 0: the paper's separate
# seed kernel.  Both must give the oracle's stream on every launch form.
FUSED_PATHS = ("ring", "time_parallel", "epoch", "chunks", "e2e", "zerocopy", "host", "device_stream")


def _run_path(path, kname, fused, output, n, i, seed, gid_begin=0, count=None):
    import torch
    count = n - gid_begin if count is None else count
    h = P.prng_create_range(n, seed, gid_begin, count)
    try:
        P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, fused)
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(kname))
        P.prng_set_option(h, P.PRNG_OPT_OUTPUT, output)
        if path == "epoch":
            P.prng_set_option(h, P.PRNG_OPT_EPOCH_ITERS, 3)
        if path == "chunks":
            P.prng_set_option(h, P.PRNG_OPT_CHUNK_ITERS, 4)
        P.prng_init(h)
        if path in ("ring", "time_parallel", "epoch", "chunks"):
            if path != "time_parallel":
                P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, i)
            P.prng_generate(h, i)
            _, _, slots, first, _ = P.prng_device_ring(h)
            out = np.stack([P.prng_read_slot(h, (first + k) % slots, count) for k in range(i)])
            vid, ep = P.prng_last_launch(h)
        elif path in ("e2e", "zerocopy"):
            P.prng_set_option(h, P.PRNG_OPT_MODE, P.PRNG_MODE_ZEROCOPY if path == "zerocopy" else P.PRNG_MODE_OVERLAP2)
            P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 3)
            out = np.zeros((i, count), np.uint64)
            P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), count, 0, i, gid_begin))
        elif path == "host":
            out = np.zeros((i, count), np.uint64)
            P.prng_generate_host(h, i, out, count, i)
        else:  # caller-owned device buffer on torch's stream
            pitch = (count + 3) // 4 * 4
            buf = torch.zeros((i, pitch), dtype=torch.int64, device="cuda")
            P.prng_generate_device(h, i, buf.data_ptr(), pitch, i, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            out = buf[:, :count].cpu().numpy().view(np.uint64).copy()
        st = P.prng_read_state(h, count)
    finally:
        P.prng_destroy(h)
    return out, st


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("path", FUSED_PATHS)
@pytest.mark.parametrize("kname", ["auto", "v4n8s1a", "v2n32s1", "v2n2s1"])
def test_fused_seed_every_launch_form(kname, path, fused):
    """Fused and separate a1 on every launch form (natural order on a ring, time-parallel
    chunks, epoch order, forced chunks, the e2e double buffer, zero-copy, the host array, a
    caller device buffer on another stream): the whole stream and the final state, vs the
    oracle, on a ragged handle with a non-zero gid offset."""
    n, gb = 9000 if path == "time_parallel" else 70001, 1233  # count 68768: 32-B rows (zero-copy), ragged pieces
    i = 700 if path == "time_parallel" else 9
    out, st = _run_path(path, kname, fused, 0, n, i, SEED_PARITY, gid_begin=gb)
    want = oracle.stream(n, i, SEED_PARITY, gb, n - gb)
    assert np.array_equal(out, want), (kname, path, fused)
    assert np.array_equal(st, want[-1])


@pytest.mark.parametrize("path", ["ring", "time_parallel", "epoch", "e2e", "host"])
def test_fused_seed_star_output(path):
    """The scrambled output (NEXT-3) starting from fused seeds (the state stays unscrambled)."""
    n, i = (5000, 600) if path == "time_parallel" else (33333, 7)
    out, st = _run_path(path, "auto", 1, 1, n, i, 77)
    assert np.array_equal(out, oracle.stream_star(n, i, 77))
    assert np.array_equal(st, oracle.stream(n, i, 77)[-1])


def test_fused_seed_read_state_right_after_init():
    """prng_read_state between prng_init and the first generate runs the pending seed
    kernel: it returns the seeds (iteration 0), and generation then continues bit-exactly;
    a second init re-arms the pending seeds."""
    n, seed = 4097, 21
    want = oracle.stream(n, 5, seed)
    h = P.prng_create(n, seed)
    try:
        P.prng_init(h)
        assert np.array_equal(P.prng_read_state(h, n), want[0])
        P.prng_generate(h, 5)
        assert np.array_equal(P.prng_read_state(h, n), want[4])
        P.prng_init(h)  # pending again: the next launch seeds in registers
        out = np.zeros((5, n), np.uint64)
        P.prng_generate(h, 5, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), n, 0, 5, 0))
        assert np.array_equal(out, want)
    finally:
        P.prng_destroy(h)


def test_fused_seed_option_roundtrip_and_errors():
    h = P.prng_create(100, 0)
    try:
        assert P.prng_get_option(h, P.PRNG_OPT_FUSED_SEED) == 1
        P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, 0)
        assert P.prng_get_option(h, P.PRNG_OPT_FUSED_SEED) == 0
        for bad in (-1, 2):
            with pytest.raises(P.PrngError) as e:
                P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, bad)
            assert e.value.code == P.PRNG_EINVAL
    finally:
        P.prng_destroy(h)


@pytest.mark.parametrize("fused", [1, 0])
def test_fused_seed_top_of_gid_range_and_a3(fused):
    """Fused seeding hashes the GLOBAL gid (gid_begin + handle-relative index) up to 2^32 - 1,
    including the A3 zero -> 1 fix-up at the derived trigger gid."""
    n = 1 << 32
    gb, cnt = A3_GID - 700, 1500
    out, st = _run_path("ring", "auto", fused, 0, n, 3, A3_SEED, gid_begin=gb, count=cnt)
    assert out[0][700] == 1
    assert np.array_equal(out, oracle.stream(n, 3, A3_SEED, gb, cnt))
    gb2 = (1 << 32) - 999
    out2, st2 = _run_path("e2e", "auto", fused, 0, n, 4, 5, gid_begin=gb2, count=999)
    want2 = oracle.stream(n, 4, 5, gb2, 999)
    assert np.array_equal(out2, want2) and np.array_equal(st2, want2[-1])


# ---------------------------------------------------------------- one-shot grids (PRNG_OPT_ONE_SHOT)
@pytest.mark.parametrize("out_kind", [0, 1])
@pytest.mark.parametrize("kname", ALL_NAMES)
def test_one_shot_every_variant(kname, out_kind):
    """PRNG_OPT_ONE_SHOT 2 forces the one-shot grid (one piece per warp, 4-warp CTAs, many
    waves) at a small ragged size: every slot of a ring that holds the whole launch and the
    state vs the oracle, for every variant and both output transforms; the grid reported by
    prng_last_grid is the one-shot one."""
    n, i = 300007, 13
    h = P.prng_create(n, SEED_PARITY)
    try:
        P.prng_set_option(h, P.PRNG_OPT_KERNEL, _kid(kname))
        P.prng_set_option(h, P.PRNG_OPT_OUTPUT, out_kind)
        P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, 2)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, i)
        P.prng_init(h)
        P.prng_generate(h, i)
        blocks, threads, rounds, os_ = P.prng_last_grid(h)
        vid, _ = P.prng_last_launch(h)
        npt = {"v4n8s1a": 8, "v4n4s1p": 4, "v4n8s1": 8, "v4n16s1": 16, "v2n32s1": 32, "v2n4s1": 4, "v4n4s1": 4,
               "v2n2s1": 2}[P.prng_kernel_variant_name(vid)]
        pieces = -(-n // (32 * npt))
        assert (os_, threads, rounds, blocks) == (True, 128, 1, -(-pieces // 4))
        _, _, slots, first, _ = P.prng_device_ring(h)
        got = np.stack([P.prng_read_slot(h, (first + k) % slots, n) for k in range(i)])
        st = P.prng_read_state(h, n)
    finally:
        P.prng_destroy(h)
    assert np.array_equal(got, (oracle.stream_star if out_kind else oracle.stream)(n, i, SEED_PARITY))
    assert np.array_equal(st, oracle.stream(n, i, SEED_PARITY)[-1])


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("path", ["e2e", "host", "device_stream", "zerocopy"])
def test_one_shot_launch_forms(path, fused):
    """One-shot grids under the other launch forms (the e2e double buffer, the host array, a
    caller device buffer on another stream, zero-copy), with fused and separate a1, on a
    gid-offset ragged handle."""
    import torch
    n, gb, i = 100001, 33, 7
    cnt = n - gb - 4   # 99964: 32-B rows for zero-copy, a ragged last piece
    h = P.prng_create_range(n, 11, gb, cnt)
    try:
        P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, 2)
        P.prng_set_option(h, P.PRNG_OPT_FUSED_SEED, fused)
        P.prng_init(h)
        if path in ("e2e", "zerocopy"):
            P.prng_set_option(h, P.PRNG_OPT_MODE, P.PRNG_MODE_ZEROCOPY if path == "zerocopy" else P.PRNG_MODE_OVERLAP2)
            P.prng_set_option(h, P.PRNG_OPT_BATCH_ITERS, 3)
            out = np.zeros((i, cnt), np.uint64)
            P.prng_generate(h, i, P.SINK_COPY, P.CopySink(out.ctypes.data_as(P.P64), cnt, 0, i, gb))
        elif path == "host":
            out = np.zeros((i, cnt), np.uint64)
            P.prng_generate_host(h, i, out, cnt, i)
        else:
            pitch = (cnt + 3) // 4 * 4
            buf = torch.zeros((i, pitch), dtype=torch.int64, device="cuda")
            P.prng_generate_device(h, i, buf.data_ptr(), pitch, i, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            out = buf[:, :cnt].cpu().numpy().view(np.uint64).copy()
        assert P.prng_last_grid(h)[3]
        st = P.prng_read_state(h, cnt)
    finally:
        P.prng_destroy(h)
    want = oracle.stream(n, i, 11, gb, cnt)
    assert np.array_equal(out, want) and np.array_equal(st, want[-1])


def test_one_shot_not_where_it_would_absorb_or_chunk():
    """The one-shot grid is not used where the rule keeps other forms: a launch that wraps a
    small ring (its resident set would rewrite L2-resident lines: the anti-absorption rule
    decides), a time-parallel launch (auto, few pieces), a user-fixed grid, forced epochs or
    chunks, or PRNG_OPT_ONE_SHOT 0."""
    cases = [  # (n, iters, ring slots, extra options, expect one-shot)
        (1 << 20, 80, 8, [(P.PRNG_OPT_ONE_SHOT, 2)], False),           # wraps 8 slots: would absorb
        (4000, 1000, 0, [], False),                                      # auto: time-parallel chunks
        (300007, 9, 9, [(P.PRNG_OPT_GRID_WARPS, 296)], False),          # user grid
        (300007, 9, 9, [(P.PRNG_OPT_EPOCH_ITERS, 3)], False),           # forced epochs
        (300007, 9, 9, [(P.PRNG_OPT_CHUNK_ITERS, 4)], False),           # forced chunks
        (300007, 9, 9, [], False),                                       # auto: < 8 waves of pieces
        (300007, 9, 9, [(P.PRNG_OPT_ONE_SHOT, 2)], True),
        (300007, 9, 9, [(P.PRNG_OPT_ONE_SHOT, 0)], False),
    ]
    for n, i, R, opts, expect in cases:
        h = P.prng_create(n, 4)
        try:
            P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, R)
            for o, v in opts:
                P.prng_set_option(h, o, v)
            P.prng_init(h)
            P.prng_generate(h, i)
            assert P.prng_last_grid(h)[3] == expect, (n, i, R, opts)
            _, _, slots, first, _ = P.prng_device_ring(h)
            assert np.array_equal(P.prng_read_slot(h, (first + i - 1) % slots, n), oracle.stream(n, i, 4)[-1])
        finally:
            P.prng_destroy(h)


def test_one_shot_option_roundtrip_and_errors():
    h = P.prng_create(100, 0)
    try:
        assert P.prng_get_option(h, P.PRNG_OPT_ONE_SHOT) == 1
        for v in (0, 2, 1):
            P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, v)
            assert P.prng_get_option(h, P.PRNG_OPT_ONE_SHOT) == v
        for bad in (-1, 3):
            with pytest.raises(P.PrngError) as e:
                P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, bad)
            assert e.value.code == P.PRNG_EINVAL
        assert P.prng_last_grid(h) == (0, 0, 0, False)
    finally:
        P.prng_destroy(h)


def test_one_shot_widens_instead_of_absorbing():
    """A wrapping launch whose default variant's one-shot resident set would rewrite
    L2-resident lines takes the narrowest wider variant that clears 2 x L2, still on the
    one-shot grid (2^20 through 40 slots, forced one-shot: v4n4s1p's 40 x 1776 x 1 KiB =
    73 MB would absorb, v4n16s1's 40 x 1776 x 4 KiB = 291 MB does not); every slot still
    held and the state vs the oracle."""
    n, i, R = 1 << 20, 100, 40
    h = P.prng_create(n, 8)
    try:
        P.prng_set_option(h, P.PRNG_OPT_ONE_SHOT, 2)
        P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, R)
        P.prng_init(h)
        P.prng_generate(h, i)
        vid, ep = P.prng_last_launch(h)
        assert (P.prng_kernel_variant_name(vid), ep) == ("v4n16s1", 0)
        assert P.prng_last_grid(h)[3]
        _, _, slots, first, _ = P.prng_device_ring(h)
        rows = {k: P.prng_read_slot(h, (first + k) % slots, n) for k in range(i - R, i)}
        st = P.prng_read_state(h, n)
    finally:
        P.prng_destroy(h)
    want = oracle.stream(n, i, 8)
    for k, row in rows.items():
        assert np.array_equal(row, want[k]), k
    assert np.array_equal(st, want[-1])
