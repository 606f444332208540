"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on identical seeded inputs.  Bar: bits, iteration
counts, flags, edge visits and BER/FER counters bit-exact; check-beliefs
(Omega) within 1e-5 absolute (observed: exact)."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

cbp = pytest.importorskip("paper_2305_05286_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module", params=[1, 2], ids=["P1", "P2"])
def fpl(request):
    """Frames per lane of the kernel geometry: every parity test runs
    with one frame per lane and with two interleaved frames per lane."""
    _need_gpu()
    return request.param


def make_code(base, Z, fpl):
    try:
        return cbp.Code(base, Z, frames_per_lane=fpl)
    except cbp.CbpError as e:
        if fpl == 2 and "two frames per lane" in str(e):
            pytest.skip("two frames per lane need the state in shared memory (Z <= 256)")
        raise


@pytest.fixture(scope="module")
def codes(fpl):
    cache = {}

    def get(name):
        if name not in cache:
            base, Z = inputs.config_base(name)
            cache[name] = (make_code(base, Z, fpl), oracle.OracleCode(base, Z))
        g = cache[name][0]
        assert g.launch_info()["frames_per_lane"] == fpl
        return cache[name]
    return get


def gpu_decode(g, llr_np, max_iter, rule=0, ld=None, omega=True, **alg):
    F, N = llr_np.shape
    ld = ld or (N + 3) // 4 * 4
    x = torch.zeros((F, ld), dtype=torch.float32)
    x[:, :N] = torch.from_numpy(llr_np)
    out = g.decode(x.cuda(), max_iter, rule, omega=omega, ev=True, **alg)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def assert_same(go, oo, N, omega=True):
    W = oo["bits"].shape[1]
    gb = go["bits"].view(np.uint32)[:, :W]
    bad = np.nonzero(~(gb == oo["bits"]).all(axis=1) | (go["iters"] != oo["iters"]) |
                     (go["flags"] != oo["flags"]) | (go["ev"] != oo["edge_visits"]))[0]
    assert len(bad) == 0, (f"{len(bad)} frames differ, first {bad[:5]}: gpu iters {go['iters'][bad[:5]]} "
                           f"oracle {oo['iters'][bad[:5]]}; flags {go['flags'][bad[:5]]} vs {oo['flags'][bad[:5]]}")
    if omega:
        np.testing.assert_allclose(go["omega"], oo["omega"], rtol=0, atol=1e-5)


# ---------------------------------------------------------------- contract bits
def test_contract_bit_equal_on_device():
    _need_gpu()
    rng = np.random.default_rng(0)
    lo, hi = np.log(1e-14), np.log(40.0)
    x = np.concatenate([np.exp(rng.uniform(lo, hi, 1 << 22)), [0.0, 1.0, 30.0, 1e-40, 1e30, np.inf]]).astype(np.float32)
    # dense exhaustive slices around the regime switch x = 2 and the clamps 30, PHI_LO
    for centre in (1.0, 2.0, 30.0, oracle.PHI_LO):
        b = np.float32(centre).view(np.uint32).astype(np.int64)
        x = np.concatenate([x, (np.arange(b - 100000, b + 100000)).astype(np.uint32).view(np.float32)])
    y_gpu = cbp.cbp.eval_contract(0, torch.from_numpy(x).cuda()).cpu().numpy()
    y_ora = oracle.phi32_array(x)
    assert (y_gpu.view(np.uint32) == y_ora.view(np.uint32)).all()
    u = (np.arange(1, 1 << 24, 7, dtype=np.float64) * 2.0 ** -24).astype(np.float32)
    assert (cbp.cbp.eval_contract(1, torch.from_numpy(u).cuda()).cpu().numpy().view(np.uint32) ==
            oracle.ln32_array(u).view(np.uint32)).all()
    m = np.arange(0, 1 << 24, 13, dtype=np.uint32)
    s_gpu = cbp.cbp.eval_contract(2, torch.from_numpy(m.view(np.float32)).cuda()).cpu().numpy()
    c_gpu = cbp.cbp.eval_contract(3, torch.from_numpy(m.view(np.float32)).cuda()).cpu().numpy()
    for k in range(0, len(m), 997):
        s, c = oracle.sincos_quarter32(int(m[k]))
        assert np.float32(s) == s_gpu[k] and np.float32(c) == c_gpu[k]


def test_phi_table_of_the_product_equals_oracle_table():
    """The v3 table is built by the product (cbp_api.cpp, host double log1p/expm1 + Newton
    differences, uploaded per device) and independently by the oracle: identical bits."""
    _need_gpu()
    g = cbp.cbp.phi_table(0).cpu().numpy()
    o = oracle.phi32_table()
    # device storage form: x < 2 segments keep c1, c2, c3 times 16, 256, 4096 (exact scaling)
    o[:704] *= np.float32([1.0, 16.0, 256.0, 4096.0])
    assert g.shape == o.shape and (g.view(np.uint32) == o.view(np.uint32)).all()


# ---------------------------------------------------------------- decode parity
def test_decode_parity_c1_all_10k_frames(codes):
    """BASELINE config 1: every one of the 10,000 frames at 2.0 dB."""
    g, o = codes("C1")
    llr, _ = o.channel(2.0, seed=1, frame_begin=0, frames=10_000)
    oo = o.decode(llr, 20, want_omega=True)
    assert_same(gpu_decode(g, llr, 20), oo, o.N)


@pytest.mark.parametrize("name,ebn0,frames", [("C2", 1.0, 400), ("C2", 2.0, 1000), ("C2", 3.0, 1000),
                                              ("C3a", 2.0, 200), ("C3a", 1.5, 100), ("C3b", 3.5, 200),
                                              ("T24", 4.0, 2000)])
def test_decode_parity_configs(codes, name, ebn0, frames):
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    llr, _ = o.channel(ebn0, seed=3, frame_begin=0, frames=frames)
    assert_same(gpu_decode(g, llr, mi), o.decode(llr, mi, want_omega=True), o.N)


@pytest.mark.parametrize("rule", [oracle.STOP_BELIEF_M, oracle.STOP_BELIEF_N, oracle.STOP_SYNDROME, oracle.STOP_NONE])
@pytest.mark.parametrize("max_iter", [1, 2, 7])
def test_decode_parity_stop_rules(codes, rule, max_iter):
    g, o = codes("C2")
    llr, _ = o.channel(2.0, seed=4, frame_begin=50, frames=200)
    assert_same(gpu_decode(g, llr, max_iter, rule), o.decode(llr, max_iter, rule, want_omega=True), o.N)


def test_decode_parity_degree_one_and_mid_row_stops(fpl):
    """C4-like degree-1 extension rows (reading R3) and many belief fires that
    fail verification (mid-row stop + rollback path, reading R5)."""
    base = inputs.construct_base((8, 14, 8, 4, 0, 3, 3), 1)
    g, o = make_code(base, 8, fpl), oracle.OracleCode(base, 8)
    for eb in (1.0, 3.0, 5.0):
        llr, _ = o.channel(eb, seed=5, frame_begin=0, frames=600)
        for rule in (0, 1, 2, 3):
            oo = o.decode(llr, 25, rule, want_omega=True)
            assert_same(gpu_decode(g, llr, 25, rule), oo, o.N)
    assert oo["fires"].sum() >= 0


def test_decode_parity_random_llrs_and_extremes(codes):
    g, o = codes("C2")
    rng = np.random.default_rng(7)
    llr = inputs.random_llr(o.N, 300, 3.0, seed=7)
    llr[0] = 0.0                                          # tie rule
    llr[1] = 1e30                                         # huge, beyond the phi clamp
    llr[2] = -1e-30
    llr[3, ::2] = np.float32(-0.0)
    llr[4] = rng.choice([-50.0, 50.0], o.N)
    assert_same(gpu_decode(g, llr, 30), o.decode(llr, 30, want_omega=True), o.N)


def test_decode_padding_and_empty(codes):
    g, o = codes("C1")
    llr, _ = o.channel(2.0, seed=2, frame_begin=0, frames=64)
    go = gpu_decode(g, llr, 20, ld=128)                   # ld > N
    assert_same(go, o.decode(llr, 20, want_omega=True), o.N)
    out = g.alloc_outputs(4)
    out["bits"] = torch.full((4, 7), -1, dtype=torch.int32, device="cuda")   # ld_words > ceil(N/32)
    g.decode(torch.from_numpy(np.ascontiguousarray(llr[:4])).cuda(), 20, out=out)
    b = out["bits"].cpu().numpy()
    assert (b[:, 3:] == 0).all()
    e = g.decode(torch.empty((0, 96), dtype=torch.float32, device="cuda"), 20)
    assert e["iters"].numel() == 0


def test_decode_i8_parity(codes):
    g, o = codes("C2")
    l8, _ = o.channel(2.5, seed=8, frame_begin=0, frames=500, llr_mode=1)
    q = np.zeros((500, 656), np.int8)
    q[:, :o.N] = np.rint(l8 * 4).astype(np.int8)
    out = g.decode_i8(torch.from_numpy(q).cuda(), 0.25, 30, omega=True, ev=True)
    torch.cuda.synchronize()
    go = {k: v.cpu().numpy() for k, v in out.items()}
    assert_same(go, o.decode(l8, 30, want_omega=True), o.N)


# ---------------------------------------------------------------- channel + ber_sim
@pytest.mark.parametrize("name,llr_mode", [("C1", 0), ("C2", 0), ("C2", 1), ("C3a", 0), ("C3b", 0)])
def test_channel_parity(codes, name, llr_mode):
    g, o = codes(name)
    for fb in (0, (1 << 32) - 3):                          # frame index across the 32-bit boundary
        l_o, cw_o = o.channel(1.5, seed=0xDEADBEEF12345678, frame_begin=fb, frames=40, llr_mode=llr_mode)
        l_g, cw_g = g.channel(1.5, seed=0xDEADBEEF12345678, frame_begin=fb, frames=40, llr_mode=llr_mode)
        assert (l_g[:, :o.N].cpu().numpy().view(np.uint32) == l_o.view(np.uint32)).all()
        assert (cw_g.cpu().numpy().view(np.uint32) == cw_o).all()


@pytest.mark.parametrize("name", ["C2", "C3a"])
def test_channel_row_pitch_and_alignment(codes, name):
    """cbp_channel with rows of ld % 4 != 0 floats and with a buffer that is only 4-byte aligned (the
    channel-only launch then stores the LLRs one by one instead of 128 bits at a time): same bits,
    and the padding columns stay untouched."""
    g, o = codes(name)
    F, N = 33, o.N
    l_o, cw_o = o.channel(2.0, seed=77, frame_begin=5, frames=F, llr_mode=0)
    for ld, off in ((N + 1, 0), (N + 4, 1), (N + 3, 3)):
        flat = torch.full((F * ld + 4,), 123.0, dtype=torch.float32, device="cuda")
        llr = flat[off:off + F * ld].view(F, ld)
        cw = torch.zeros((F, g.words), dtype=torch.int32, device="cuda")
        g.channel(2.0, seed=77, frame_begin=5, frames=F, llr_mode=0, out=(llr, cw))
        torch.cuda.synchronize()
        got = llr.cpu().numpy()
        assert (got[:, :N].view(np.uint32) == l_o.view(np.uint32)).all(), (ld, off)
        assert (got[:, N:] == 123.0).all(), (ld, off)
        assert (cw.cpu().numpy().view(np.uint32) == cw_o).all()


@pytest.mark.parametrize("name,ebn0,frames,llr_mode", [("C1", 2.0, 10_000, 0), ("C2", 1.5, 1500, 0),
                                                       ("C2", 2.5, 1500, 1), ("C3a", 2.5, 200, 0),
                                                       ("C3b", 4.0, 200, 0)])
def test_ber_sim_parity(codes, name, ebn0, frames, llr_mode):
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    want = o.ber_sim(ebn0, 21, 1000, frames, mi, llr_mode=llr_mode)
    got = g.ber_sim(ebn0, 21, 1000, frames, mi, llr_mode=llr_mode).cpu().numpy()
    assert list(got) == list(want), dict(zip(oracle.COUNT_NAMES, zip(got, want)))


def test_ber_sim_full_size_sampled(codes):
    """BASELINE config 2 at full size (10^6 frames, 2.0 dB) in the bench launch
    configuration: counters equal channel -> decode -> compare on the GPU, shard
    invariant, and a seeded sample of frames (plus error frames) equal the oracle."""
    g, o = codes("C2")
    F, seed, eb = 1_000_000, 1, 2.0
    full = g.ber_sim(eb, seed, 0, F, 30).cpu().numpy()
    halves = (g.ber_sim(eb, seed, 0, 400_000, 30) + g.ber_sim(eb, seed, 400_000, F - 400_000, 30)).cpu().numpy()
    assert (full == halves).all()
    # channel -> decode on the GPU reproduces the fused counters
    tot = np.zeros(8, np.int64)
    err_frames = []
    for b in range(0, F, 250_000):
        llr, cw = g.channel(eb, seed, b, 250_000)
        out = g.decode(llr, 30, ev=True)
        d = cbp.unpack_bits(out["bits"], o.N) != cbp.unpack_bits(cw, o.N)
        info = d[:, :o.K].sum(1)
        tot += np.array([250_000, info.sum().item(), (info > 0).sum().item(), d.any(1).sum().item(),
                         out["iters"].sum().item(), out["ev"].sum().item(),
                         ((out["flags"] & 1) == 0).sum().item(), 0], np.int64)
        err_frames += (b + torch.nonzero((info > 0) | ((out["flags"] & 1) == 0)).flatten().cpu().numpy()).tolist()
    assert (tot[:7] == full[:7]).all()
    rng = np.random.default_rng(3)
    sample = sorted(set(rng.integers(0, F, 150).tolist() + err_frames[:100]))
    for fidx in sample:
        llr_o, _ = o.channel(eb, seed, fidx, 1)
        llr_g, _ = g.channel(eb, seed, fidx, 1)
        assert (llr_g[:, :o.N].cpu().numpy() == llr_o).all()
        assert_same(gpu_decode(g, llr_o, 30), o.decode(llr_o, 30, want_omega=True), o.N)


# ---------------------------------------------------------------- C4: Z = 384, state in global memory
@pytest.mark.parametrize("rule", [oracle.STOP_SYNDROME, oracle.STOP_BELIEF_M])
def test_c4_decode_parity(codes, rule):
    """BASELINE config 4 (N=26112, 42 degree-1 extension columns): one frame per CTA on
    cbp_warp_kernel's team path (Lambda and the H bytes, 130 KB, in shared memory; 12 warps
    ordered by a CTA barrier per row); with the Omega output (S, 70 KB more) the frame moves to
    cbp_kernel's L2-resident global workspace.  Both equal the oracle."""
    g, o = codes("C4")
    li = g.launch_info()
    assert li["state_in_smem"] == 1 and li["threads"] == 384 and li["frames_per_cta"] == 1, li
    llr, _ = o.channel(1.5, seed=12, frame_begin=0, frames=6)
    want = o.decode(llr, 25, rule, want_omega=True)
    assert_same(gpu_decode(g, llr, 25, rule), want, o.N)
    assert_same(gpu_decode(g, llr, 25, rule, omega=False), want, o.N, omega=False)


@pytest.mark.parametrize("env", [{}, {"CBP_WARP_TEAM": "0"}], ids=["team", "cbp_kernel"])
@pytest.mark.parametrize("name,eb,frames,mi", [("C4", 1.5, 5, 12), ("P8192", 1.5, 24, 20), ("C3a", 2.0, 150, 30)])
def test_team_frames_equal_oracle(monkeypatch, env, name, eb, frames, mi):
    """Team frames (one frame per CTA) -- the automatic geometry of C4 and P8192 --
    and, forced with CBP_WARP_TEAM=0, cbp_kernel's teams for the same codes: decode (no Omega, the
    team path) and ber_sim (fp32 and int8 streams) equal the oracle frame by frame / counter by
    counter.  C3a (warp mode) runs as a control."""
    _need_gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    base, Z = inputs.config_base(name)
    g, o = cbp.Code(base, Z), oracle.OracleCode(base, Z)
    lm = 2 if inputs.is_peg(name) else 0
    llr, _ = o.channel(eb, seed=31, frame_begin=0, frames=frames, llr_mode=lm)
    for rule in (oracle.STOP_BELIEF_M, oracle.STOP_SYNDROME):
        assert_same(gpu_decode(g, llr, mi, rule, omega=False), o.decode(llr, mi, rule), o.N, omega=False)
    for llr_mode in ((2,) if inputs.is_peg(name) else (0, 1)):
        want = o.ber_sim(eb, 9, 0, frames, mi, llr_mode=llr_mode)
        got = g.ber_sim(eb, 9, 0, frames, mi, llr_mode=llr_mode).cpu().numpy()
        assert list(got) == list(want), (llr_mode, list(got), list(want))


def test_c4_ber_sim_parity(codes):
    g, o = codes("C4")
    want = o.ber_sim(2.0, 5, 0, 6, 25, stop_rule=oracle.STOP_SYNDROME)
    got = g.ber_sim(2.0, 5, 0, 6, 25, stop_rule=oracle.STOP_SYNDROME).cpu().numpy()
    assert list(got) == list(want)


# ---------------------------------------------------------------- NEXT-1: normalized min-sum CBP
MS = dict(algorithm=1)


@pytest.mark.parametrize("name,ebn0,frames,alpha", [("C1", 2.0, 3000, 0.75), ("C2", 2.0, 1000, 0.75),
                                                    ("C2", 1.5, 500, 1.0), ("C2", 3.0, 500, 0.625),
                                                    ("C3a", 2.0, 150, 0.75), ("C3b", 3.5, 150, 0.8),
                                                    ("T24", 4.0, 1000, 0.75)])
def test_minsum_decode_parity(codes, name, ebn0, frames, alpha):
    """Normalized min-sum CBP (reading R20) on the GPU equals
    the oracle's min-sum CBP bit for bit, Omega = sgn * min included."""
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    llr, _ = o.channel(ebn0, seed=31, frame_begin=0, frames=frames)
    oo = o.decode(llr, mi, want_omega=True, arith=oracle.MINSUM, alpha=alpha)
    go = gpu_decode(g, llr, mi, alpha=alpha, **MS)
    assert_same(go, oo, o.N, omega=False)
    assert (go["omega"].view(np.uint32) == oo["omega"].view(np.uint32)).all()


@pytest.mark.parametrize("rule", [oracle.STOP_BELIEF_M, oracle.STOP_BELIEF_N, oracle.STOP_SYNDROME, oracle.STOP_NONE])
def test_minsum_stop_rules_and_extremes(codes, rule):
    g, o = codes("C2")
    llr = inputs.random_llr(o.N, 200, 2.5, seed=9)
    llr[0] = 0.0
    llr[1] = 1e30
    llr[2, ::3] = np.float32(-0.0)
    llr[3] = np.where(np.arange(o.N) % 2 == 0, 4.0, -4.0)      # many equal magnitudes: owner ties
    for mi in (1, 7):
        oo = o.decode(llr, mi, rule, oracle.MINSUM, want_omega=True, alpha=0.75)
        go = gpu_decode(g, llr, mi, rule, alpha=0.75, **MS)
        assert_same(go, oo, o.N, omega=False)
        assert (go["omega"].view(np.uint32) == oo["omega"].view(np.uint32)).all()


def test_minsum_multi_warp_team_and_global_state(codes, fpl):
    """Z > 32 (multi-warp teams) and Z = 384 with the state in global memory."""
    base = inputs.construct_base((6, 18, 96, 6, 1, 2, 4), 2)
    g2, o2 = make_code(base, 96, fpl), oracle.OracleCode(base, 96)
    llr, _ = o2.channel(2.0, seed=14, frame_begin=0, frames=60)
    for rule in (0, 2):
        oo = o2.decode(llr, 15, rule, oracle.MINSUM, want_omega=True, alpha=0.75)
        assert_same(gpu_decode(g2, llr, 15, rule, alpha=0.75, **MS), oo, o2.N)
    g, o = codes("C4")
    llr, _ = o.channel(1.5, seed=13, frame_begin=0, frames=4)
    oo = o.decode(llr, 20, oracle.STOP_SYNDROME, oracle.MINSUM, want_omega=True, alpha=0.75)
    assert_same(gpu_decode(g, llr, 20, oracle.STOP_SYNDROME, alpha=0.75, **MS), oo, o.N, omega=False)


@pytest.mark.parametrize("name,ebn0,frames,llr_mode", [("C2", 2.0, 2000, 0), ("C2", 2.5, 1000, 1),
                                                       ("C3a", 2.5, 150, 0)])
def test_minsum_ber_sim_parity(codes, name, ebn0, frames, llr_mode):
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    want = o.ber_sim(ebn0, 23, 500, frames, mi, llr_mode=llr_mode, arith=oracle.MINSUM, alpha=0.75)
    got = g.ber_sim(ebn0, 23, 500, frames, mi, llr_mode=llr_mode, alpha=0.75, **MS).cpu().numpy()
    assert list(got) == list(want), dict(zip(oracle.COUNT_NAMES, zip(got, want)))


def test_minsum_rejects_bad_options(codes, fpl):
    g, o = codes("C2")
    x = torch.zeros((2, 648), dtype=torch.float32, device="cuda")
    for a in (0.0, -0.5, 1.5, float("nan")):
        with pytest.raises(RuntimeError):
            g.decode(x, 5, alpha=a, **MS)
    with pytest.raises(RuntimeError):
        g.decode(x, 5, algorithm=7)
    # a degree-1 check row has no leave-one-out minimum: min-sum is refused, log-tanh decodes
    base = np.array([[0, 1, -1, 2], [-1, 2, 0, -1], [-1, -1, 3, -1]], np.int16)   # last base row: degree 1
    g1 = make_code(base, 8, fpl)
    y = torch.zeros((2, 32), dtype=torch.float32, device="cuda")
    g1.decode(y, 5)
    with pytest.raises(RuntimeError):
        g1.decode(y, 5, **MS)


def test_decode_host_pipeline(codes):
    """The end-to-end path of bench.py's e2e (pinned host LLRs -> chunked H2D / cbp_decode
    / D2H over several streams) returns exactly the device-resident decode's outputs,
    for a frame count that leaves a ragged last chunk; a sample equals the oracle."""
    from paper_2305_05286_b200 import pipeline
    g, o = codes("C2")
    F = 3 * (1 << 15) + 777
    llr, _ = g.channel(2.0, 17, 0, F, want_cw=False)
    host = torch.empty(tuple(llr.shape), dtype=torch.float32, pin_memory=True)
    host.copy_(llr)
    out = pipeline.decode_host(g, host, 30)
    ref = g.decode(llr, 30)
    torch.cuda.synchronize()
    for k in ("bits", "iters", "flags"):
        assert torch.equal(out[k], ref[k].cpu()), k
    idx = np.array([0, 1, F // 2, F - 1])
    l_o = llr[idx].cpu().numpy()[:, :o.N]
    oo = o.decode(np.ascontiguousarray(l_o), 30)
    assert (out["bits"].numpy()[idx].view(np.uint32)[:, :oo["bits"].shape[1]] == oo["bits"]).all()
    assert (out["iters"].numpy()[idx] == oo["iters"]).all()


def test_decode_host_abi_int8_and_errors(codes):
    """cbp_decode_host_i8 (host int8 LLRs) equals the device decode; chunk / stream settings do
    not change results; the host entry points reject bad arguments without touching outputs,
    and the binding rejects undersized output buffers (the ABI cannot see their sizes)."""
    import ctypes
    g, o = codes("C2")
    F = 5000
    llr, _ = g.channel(2.0, 21, 0, F, llr_mode=1, want_cw=False)
    q = torch.round(llr * 4).clamp(-127, 127).to(torch.int8)
    ldq = (g.N + 15) // 16 * 16
    qh = torch.zeros((F, ldq), dtype=torch.int8, pin_memory=True)
    qh[:, :g.N].copy_(q[:, :g.N])
    ref = g.decode_i8(qh.cuda(), 0.25, 30)
    for chunk, ns in ((0, 0), (777, 3), (F, 1)):
        out = g.decode_host(qh, 30, scale=0.25, chunk_frames=chunk, nstreams=ns)
        for k in ("bits", "iters", "flags"):
            assert torch.equal(out[k], ref[k].cpu()), (k, chunk, ns)
    L = cbp.lib()
    ok = cbp.cbp._Opts(30, 0, 0, 0.75)
    hb = torch.zeros((F, g.words), dtype=torch.int32)
    hi = torch.full((F,), -7, dtype=torch.int32)
    hf = torch.zeros(F, dtype=torch.uint8)
    lh = torch.zeros((F, 648), dtype=torch.float32)

    def call(ld=648, frames=F, lw=g.words, chunk=0, ns=0, ptr=True):
        return L.cbp_decode_host(g.handle, lh.data_ptr() if ptr else None, ld, frames, ctypes.byref(ok),
                                 hb.data_ptr(), lw, hi.data_ptr(), hf.data_ptr(), chunk, ns)
    assert call(ld=640) == 1 and call(ld=650) == 1 and call(frames=-1) == 1 and call(lw=g.words - 1) == 1
    assert call(chunk=-1) == 1 and call(ns=17) == 1 and call(ptr=False) == 1
    assert (hi == -7).all()                                  # nothing ran
    assert call(frames=0) == 0
    with pytest.raises(cbp.CbpError):
        g.decode(llr, 30, out=g.alloc_outputs(F - 1))        # too few rows for the batch
    with pytest.raises(cbp.CbpError):
        g.ber_sim(2.0, 1, 0, 10, 30, counts=torch.zeros(4, dtype=torch.int64, device=g.device))


# ---------------------------------------------------------------- NEXT-3: comparison schedules
BP_ALGS = [(2, oracle.LBP), (3, oracle.FBP)]


@pytest.mark.parametrize("alg,arith", BP_ALGS, ids=["LBP", "FBP"])
@pytest.mark.parametrize("name,ebn0,frames", [("C1", 2.0, 2000), ("C2", 2.0, 600), ("C2", 1.0, 200),
                                              ("C3a", 2.0, 100), ("C3b", 3.5, 100), ("T24", 4.0, 500)])
def test_bp_schedule_decode_parity(codes, alg, arith, name, ebn0, frames):
    """Layered and flooding BP (the paper's comparison schedules, reading R22) on the
    GPU equal the oracle's fp32 LBP / FBP bit for bit: decisions, iterations, flags,
    edge visits, for the syndrome stop and for a fixed number of sweeps."""
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    llr, _ = o.channel(ebn0, seed=41, frame_begin=0, frames=frames)
    for rule, m in ((oracle.STOP_SYNDROME, mi), (oracle.STOP_NONE, 3)):
        oo = o.decode(llr, m, rule, arith)
        go = gpu_decode(g, llr, m, rule, algorithm=alg)
        assert_same(go, oo, o.N, omega=False)


@pytest.mark.parametrize("alg,arith", BP_ALGS, ids=["LBP", "FBP"])
def test_bp_schedule_degree_one_and_global_state(codes, fpl, alg, arith):
    base = inputs.construct_base((8, 14, 8, 4, 0, 3, 3), 1)
    g, o = make_code(base, 8, fpl), oracle.OracleCode(base, 8)
    llr, _ = o.channel(3.0, seed=42, frame_begin=0, frames=400)
    assert_same(gpu_decode(g, llr, 25, oracle.STOP_SYNDROME, algorithm=alg),
                o.decode(llr, 25, oracle.STOP_SYNDROME, arith), o.N, omega=False)
    g, o = codes("C4")
    llr, _ = o.channel(1.5, seed=43, frame_begin=0, frames=4)
    assert_same(gpu_decode(g, llr, 10, oracle.STOP_SYNDROME, algorithm=alg),
                o.decode(llr, 10, oracle.STOP_SYNDROME, arith), o.N, omega=False)


@pytest.mark.parametrize("alg,arith", BP_ALGS, ids=["LBP", "FBP"])
@pytest.mark.parametrize("name,ebn0,frames,llr_mode", [("C2", 2.0, 1500, 0), ("C2", 2.5, 800, 1), ("C3a", 2.5, 100, 0)])
def test_bp_schedule_ber_sim_parity(codes, alg, arith, name, ebn0, frames, llr_mode):
    g, o = codes(name)
    mi = inputs.CONFIGS[name].max_iter
    want = o.ber_sim(ebn0, 44, 100, frames, mi, oracle.STOP_SYNDROME, llr_mode, arith=arith)
    got = g.ber_sim(ebn0, 44, 100, frames, mi, oracle.STOP_SYNDROME, llr_mode, algorithm=alg).cpu().numpy()
    assert list(got) == list(want), dict(zip(oracle.COUNT_NAMES, zip(got, want)))


def test_bp_schedule_rejects_belief_rules(codes):
    g, o = codes("C2")
    x = torch.zeros((2, 648), dtype=torch.float32, device="cuda")
    for alg in (2, 3):
        for rule in (0, 1):
            with pytest.raises(RuntimeError):
                g.decode(x, 5, rule, algorithm=alg)
    with pytest.raises(RuntimeError):
        g.decode(x, 5, 2, algorithm=4)


def test_sweep_gpu_runner_resume(codes, tmp_path):
    """paper_2305_05286_b200.sweep with the product runner (cbp_ber_sim): chunked and
    resumed totals equal one fused launch over the whole frame range."""
    from paper_2305_05286_b200.sweep import gpu_runner, run_sweep
    g, o = codes("C2")
    run = gpu_runner(g, 30, 5)
    hdr = {"config": "C2", "seed": 5}
    out = tmp_path / "s.jsonl"
    run_sweep(run, [2.0], 150_000, 40_000, hdr, out)
    lines = out.read_text().splitlines()
    out.write_text("\n".join(lines[:-2]) + "\n")                 # drop the last two chunks: resume redoes them
    res = run_sweep(run, [2.0, 2.5], 150_000, 40_000, hdr, out)
    for eb in (2.0, 2.5):
        want = g.ber_sim(eb, 5, 0, 150_000, 30).cpu().numpy()
        c = res[eb]["counts"]
        assert [c[k] for k in cbp.COUNT_NAMES] == list(want)


def _fused_vs_unfused(g, eb, seed, begin, frames, mi, chunk, llr_mode=0):
    """channel -> (int8) decode -> compare on the GPU, chunk by chunk: the counters the fused
    ber_sim must reproduce, plus the indices of the frames with errors / no convergence."""
    tot = np.zeros(8, np.int64)
    bad = []
    for b in range(begin, begin + frames, chunk):
        n = min(chunk, begin + frames - b)
        llr, cw = g.channel(eb, seed, b, n, llr_mode=llr_mode)
        if llr_mode:
            q = torch.zeros((n, (g.N + 15) // 16 * 16), dtype=torch.int8, device=llr.device)
            q[:, :g.N] = torch.round(llr[:, :g.N] * 4).to(torch.int8)
            out = g.decode_i8(q, 0.25, mi, ev=True)
        else:
            out = g.decode(llr, mi, ev=True)
        d = cbp.unpack_bits(out["bits"], g.N) != cbp.unpack_bits(cw, g.N)
        info = d[:, :g.K].sum(1)
        tot += np.array([n, info.sum().item(), (info > 0).sum().item(), d.any(1).sum().item(),
                         out["iters"].sum().item(), out["ev"].sum().item(),
                         ((out["flags"] & 1) == 0).sum().item(), 0], np.int64)
        bad += (b + torch.nonzero((info > 0) | ((out["flags"] & 1) == 0)).flatten().cpu().numpy()).tolist()
    return tot, bad


@pytest.mark.parametrize("name,eb,begin,frames,llr_mode", [
    ("C3a", 1.5, 0, 10_000_000, 0),                       # BASELINE configs[2]: 10^7 frames per point
    ("C5", 2.5, 1_000_000_000 - 20_000_000, 20_000_000, 1)])   # configs[4]: the top slice of 10^9, int8 stream
def test_ber_sim_full_size_sampled_c3(codes, name, eb, begin, frames, llr_mode):
    """Full-size fused ber_sim in the bench launch configuration for the N=1944 code:
    shard invariance, the fused counters reproduced by channel -> decode -> compare on
    the GPU (first 10^6 frames of the range), and sampled plus error frames equal the
    oracle frame by frame."""
    g, o = codes("C3a")
    mi = 30
    full = g.ber_sim(eb, 1, begin, frames, mi, llr_mode=llr_mode).cpu().numpy()
    cut = frames // 3
    parts = (g.ber_sim(eb, 1, begin, cut, mi, llr_mode=llr_mode) +
             g.ber_sim(eb, 1, begin + cut, frames - cut, mi, llr_mode=llr_mode)).cpu().numpy()
    assert (full == parts).all() and full[0] == frames
    sub = 1_000_000
    want = g.ber_sim(eb, 1, begin, sub, mi, llr_mode=llr_mode).cpu().numpy()
    tot, bad = _fused_vs_unfused(g, eb, 1, begin, sub, mi, 250_000, llr_mode)
    assert (tot[:7] == want[:7]).all(), (tot, want)
    rng = np.random.default_rng(4)
    sample = sorted(set((begin + rng.integers(0, sub, 40)).tolist() + bad[:40]))
    for fidx in sample:
        llr_o, _ = o.channel(eb, 1, fidx, 1, llr_mode=llr_mode)
        llr_g, _ = g.channel(eb, 1, fidx, 1, llr_mode=llr_mode)
        assert (llr_g[:, :o.N].cpu().numpy() == llr_o).all()
        assert_same(gpu_decode(g, llr_o, mi), o.decode(llr_o, mi, want_omega=True), o.N)


def test_abi_error_paths(codes):
    """The documented error behaviour of include/cbp.h: every invalid argument returns
    CBP_E_INVALID (1) / CBP_E_UNSUPPORTED (2) with a message and launches nothing."""
    import ctypes
    L = cbp.lib()
    g, o = codes("C2")
    h = g.handle
    dev = torch.device("cuda", 0)
    x = torch.zeros((4, 648), dtype=torch.float32, device=dev)
    bits = torch.zeros((4, 21), dtype=torch.int32, device=dev)
    it = torch.zeros(4, dtype=torch.int32, device=dev)
    fl = torch.zeros(4, dtype=torch.uint8, device=dev)
    ok = cbp.cbp._Opts(30, 0, 0, 0.75)

    def dec(ptr=None, ld=648, frames=4, opts=ok, lw=21, b=bits):
        return L.cbp_decode(h, x.data_ptr() if ptr is None else ptr, ld, frames, ctypes.byref(opts),
                            b.data_ptr() if b is not None else None, lw, it.data_ptr(), fl.data_ptr(), None, None,
                            None)
    assert dec() == 0
    assert dec(ld=640) == 1                                    # ld < N
    assert dec(ld=650) == 1                                    # ld * 4 not a multiple of 16
    assert dec(ptr=x.data_ptr() + 4) == 1                      # misaligned input
    assert dec(frames=-1) == 1
    assert dec(lw=20) == 1                                     # ld_words < ceil(N/32)
    assert dec(b=None) == 1                                    # null output
    assert dec(frames=0, b=None) == 0                          # empty batch is a no-op
    for bad in ((0, 0, 0, 0.75), (70000, 0, 0, 0.75), (5, 4, 0, 0.75), (5, 0, 4, 0.75), (5, 0, 1, 0.0),
                (5, 0, 2, 0.75), (5, 1, 3, 0.75)):
        assert dec(opts=cbp.cbp._Opts(*bad)) == 1, bad
    assert b"opts" in L.cbp_last_error() or b"stop" in L.cbp_last_error()
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    assert L.cbp_ber_sim(h, 2.0, 1, 0, 10, ctypes.byref(ok), 4, cnt.data_ptr(), None) == 1   # llr_mode
    assert L.cbp_ber_sim(h, 2.0, 1, 0, 10, ctypes.byref(ok), -1, cnt.data_ptr(), None) == 1
    assert L.cbp_ber_sim(h, float("nan"), 1, 0, 10, ctypes.byref(ok), 0, cnt.data_ptr(), None) == 1
    assert L.cbp_ber_sim(h, 2.0, 1, -1, 10, ctypes.byref(ok), 0, cnt.data_ptr(), None) == 1
    assert L.cbp_ber_sim(h, 2.0, 1, 0, 10, ctypes.byref(ok), 0, None, None) == 1
    assert int(cnt.sum()) == 0                                 # nothing ran

    def create(base, Z, fpl=0):
        hh = ctypes.c_void_p()
        b = np.ascontiguousarray(base, np.int16)
        cfg = cbp.cbp._CodeConfig(fpl)
        rc = L.cbp_code_create_ex(b.ctypes.data, b.shape[0], b.shape[1], Z, 0, ctypes.byref(cfg), ctypes.byref(hh))
        if rc == 0:
            L.cbp_code_destroy(hh)
        return rc
    good = np.array([[0, 1, 0, -1], [2, -1, 0, 0]], np.int16)
    assert create(good, 4) == 0
    assert create(good, 0) == 1 and create(good, 1025) == 1  # Z range
    assert create(np.array([[0, 5, 0, -1], [2, -1, 0, 0]]), 4) == 1       # shift >= Z
    assert create(np.array([[0, -1, 0, -1], [2, -1, 0, 0]]), 4) == 1      # empty column
    assert create(np.array([[-1, -1, -1, -1], [2, 1, 0, 0]]), 4) == 1     # empty row
    assert create(good, 4, fpl=3) == 1                                    # frames_per_lane
    assert create(np.zeros((2, 70), np.int16), 1000) == 2                 # N >= 65536: unsupported
    assert create(np.zeros((1, 40), np.int16), 4) == 2                    # base row degree > 32
    # encoding needs the dual-diagonal structure: this base decodes but cannot simulate
    gg = cbp.Code(good, 4)
    with pytest.raises(cbp.CbpError):
        gg.ber_sim(2.0, 1, 0, 10, 5)
    gg.decode(torch.zeros((2, 16), dtype=torch.float32, device=dev), 5)


@pytest.mark.parametrize("name", ["C2", "C3a", "C3b"])
def test_ber_sim_all_frames_equal_oracle_counts(codes, name):
    """BASELINE configs[1] exactly as bench.py runs it (C2, 1.0..3.0 dB, 10^6 frames per
    point, seed 1, max_iter 30), and configs[2] (C3a at 2.5 dB, C3b at 4.0 dB, all 10^7 frames): the fused
    GPU counters over EVERY frame equal the CPU oracle's (tests/golden/oracle_counts_<name>.json,
    written by tools/write_oracle_counts.py from oracle/ alone) -- bit errors, frame errors,
    iteration and edge-visit sums."""
    import json
    from pathlib import Path
    path = Path(__file__).parent / "golden" / f"oracle_counts_{name}.json"
    if not path.exists():
        pytest.skip(f"{path.name} not written")
    gold = json.loads(path.read_text())
    g, o = codes(name)
    F = gold["frames_per_point"]
    for eb, want in gold["counts"].items():
        got = g.ber_sim(float(eb), gold["seed"], 0, F, gold["max_iter"]).cpu().numpy()
        assert list(got) == want, (eb, dict(zip(oracle.COUNT_NAMES, zip(got, want))))


def test_concurrent_streams_and_threads(codes):
    """A cbp_code is shared by several host threads and streams (include/cbp.h): concurrent
    decodes and ber_sims on four streams from four threads give the sequential results."""
    import threading
    g, o = codes("C2")
    llr, _ = g.channel(2.0, 3, 0, 20_000, want_cw=False)
    ref = g.decode(llr, 30, ev=True)
    ref_c = g.ber_sim(2.5, 9, 0, 30_000, 30).cpu()
    torch.cuda.synchronize()
    outs, cnts, errs = [None] * 4, [None] * 4, []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs[k] = g.decode(llr, 30, ev=True, stream=s)
                cnts[k] = g.ber_sim(2.5, 9, 0, 30_000, 30, stream=s)
            s.synchronize()
        except Exception as e:   # pragma: no cover
            errs.append(e)
    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(4):
        for key in ("bits", "iters", "flags", "ev"):
            assert torch.equal(outs[k][key], ref[key]), (k, key)
        assert torch.equal(cnts[k].cpu(), ref_c)


@pytest.mark.parametrize("alg,arith", [(1, oracle.MINSUM), (2, oracle.LBP), (3, oracle.FBP)],
                         ids=["min-sum", "LBP", "FBP"])
def test_decode_i8_other_algorithms(codes, alg, arith):
    """cbp_decode_i8 (int8 LLR stream, L = q/4) with the min-sum CBP and the comparison
    schedules equals the oracle on the dequantised LLRs."""
    g, o = codes("C2")
    l8, _ = o.channel(2.0, seed=51, frame_begin=0, frames=400, llr_mode=1)
    q = np.zeros((400, 656), np.int8)
    q[:, :o.N] = np.rint(l8 * 4).astype(np.int8)
    rule = oracle.STOP_BELIEF_M if alg == 1 else oracle.STOP_SYNDROME
    out = g.decode_i8(torch.from_numpy(q).cuda(), 0.25, 30, rule, ev=True, omega=True, algorithm=alg)
    torch.cuda.synchronize()
    go = {k: v.cpu().numpy() for k, v in out.items()}
    assert_same(go, o.decode(l8, 30, rule, arith, want_omega=True), o.N, omega=False)


def test_decode_deterministic_under_rescheduling(codes):
    """Race-detection substitute (compute-sanitizer is unavailable on the pool): per-frame
    results do not depend on how the persistent grid's work queue hands frames to teams --
    the same frames decoded in one launch, in uneven slices, and repeatedly, give
    identical bits, iterations, flags, edge visits and check-beliefs."""
    g, o = codes("C2")
    llr, _ = g.channel(1.5, 77, 0, 30_000, want_cw=False)
    full = g.decode(llr, 30, omega=True, ev=True)
    parts = [g.decode(llr[a:b].contiguous(), 30, omega=True, ev=True)
             for a, b in ((0, 1), (1, 4097), (4097, 4100), (4100, 30_000))]
    again = g.decode(llr, 30, omega=True, ev=True)
    torch.cuda.synchronize()
    for k in ("bits", "iters", "flags", "ev", "omega"):
        cat = torch.cat([p[k] for p in parts])
        assert torch.equal(full[k], cat), k
        assert torch.equal(full[k], again[k]), k


@pytest.mark.parametrize("spec,seed,Z,frames,eb", [
    ((3, 6, 1024, 3, 0, 3, 3), 2, 1024, 6, 2.5),        # Z = 1024: 32-warp teams (the 1024-thread instantiation)
    ((4, 36, 4, 4, 0, 3, 3), 3, 4, 200, 4.0),            # rate 8/9: base rows of degree ~28 (near max_dc = 32)
    ((60, 120, 4, 60, 0, 3, 3), 4, 4, 100, 3.0),         # 60 base rows, 120 columns
])
def test_decode_parity_size_limits(fpl, spec, seed, Z, frames, eb):
    """Codes at the ABI's limits (include/cbp.h: Z <= 1024, base row degree <= 32, many
    rows): decode and ber_sim parity with the oracle for every algorithm that applies."""
    base = inputs.construct_base(spec, seed)
    g, o = make_code(base, Z, fpl), oracle.OracleCode(base, Z)
    assert g.launch_info()["frames_per_cta"] >= 1
    llr, _ = o.channel(eb, seed=60 + seed, frame_begin=0, frames=frames)
    assert_same(gpu_decode(g, llr, 12), o.decode(llr, 12, want_omega=True), o.N)
    assert_same(gpu_decode(g, llr, 12, oracle.STOP_SYNDROME, algorithm=2),
                o.decode(llr, 12, oracle.STOP_SYNDROME, oracle.LBP), o.N, omega=False)
    want = o.ber_sim(eb, 61, 0, frames, 12)
    got = g.ber_sim(eb, 61, 0, frames, 12).cpu().numpy()
    assert list(got) == list(want)


@pytest.mark.parametrize("env", [{"CBP_SPLIT_R": "1"}, {"CBP_SPLIT_R": "0"}, {"CBP_GLOBAL_TEAMS": "8"},
                                 {"CBP_GLOBAL_TEAMS": "3"}, {"CBP_WARP_KERNEL": "0"},
                                 {"CBP_WARP_KERNEL": "0", "CBP_SPLIT_R": "1"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("name,eb,frames", [("C2", 2.0, 1500), ("C3a", 2.0, 200), ("C1", 2.0, 3000),
                                            ("P2048", 1.5, 300)])
def test_state_layouts_equal_oracle(monkeypatch, env, name, eb, frames):
    """Every state layout the geometry can pick on the same frames: all in
    shared memory, the split layout (R in the global workspace), and the all-global
    workspace with warp teams and multi-warp teams (forced through the A/B switches,
    read when a code is created): decode and ber_sim results equal the oracle's."""
    _need_gpu()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    base, Z = inputs.config_base(name)
    g, o = cbp.Code(base, Z), oracle.OracleCode(base, Z)
    info = g.launch_info()
    if "CBP_GLOBAL_TEAMS" in env:
        assert info["state_in_smem"] == 0 and info["r_in_global"] == 0
    if env.get("CBP_SPLIT_R") == "1":
        assert info["state_in_smem"] == 1 and info["r_in_global"] == 1
    if env.get("CBP_SPLIT_R") == "0":
        assert info["r_in_global"] == 0
    mi = inputs.get_config(name).max_iter
    lm = oracle.TX_ZERO if inputs.is_peg(name) else 0
    llr, _ = o.channel(eb, 9, 0, frames, llr_mode=lm)
    assert_same(gpu_decode(g, llr, mi), o.decode(llr, mi, want_omega=True), o.N)
    assert_same(gpu_decode(g, llr, mi, algorithm=1), o.decode(llr, mi, arith=oracle.MINSUM, want_omega=True),
                o.N, omega=False)
    got = g.ber_sim(eb, 12, 100, frames, mi, llr_mode=lm).cpu().numpy()
    assert list(got) == list(o.ber_sim(eb, 12, 100, frames, mi, llr_mode=lm))
    got = g.ber_sim(eb, 12, 100, frames // 2, mi, 2, llr_mode=lm, algorithm=3).cpu().numpy()
    assert list(got) == list(o.ber_sim(eb, 12, 100, frames // 2, mi, 2, llr_mode=lm, arith=oracle.FBP))


# ---------------------------------------------------------------- split ber_sim: cbp_channel + cbp_ber_count
@pytest.fixture(scope="module")
def auto_codes():
    """Codes in the default (automatic) geometry -- the one bench.py and cbp_ber_sim run."""
    _need_gpu()
    cache = {}

    def get(name):
        if name not in cache:
            base, Z = inputs.config_base(name)
            cache[name] = (cbp.Code(base, Z), oracle.OracleCode(base, Z))
        return cache[name]
    return get


@pytest.mark.parametrize("name,ebn0,frames,llr_mode,alg", [
    ("C2", 1.5, 1500, 0, 0), ("C2", 2.5, 1500, 1, 0), ("C3a", 2.5, 300, 0, 0), ("C3b", 4.0, 200, 1, 0),
    ("C2", 2.0, 600, 0, 2)])
def test_ber_count_parity(auto_codes, name, ebn0, frames, llr_mode, alg):
    """cbp_ber_count on cbp_channel's frames (the two halves of the split cbp_ber_sim) equals the
    oracle's ber_sim counters; so does cbp_ber_sim itself (split by default on these codes)."""
    g, o = auto_codes(name)
    mi = inputs.CONFIGS[name].max_iter
    rule = oracle.STOP_SYNDROME if alg == 2 else oracle.STOP_BELIEF_M
    kw = dict(arith=oracle.LBP) if alg == 2 else {}
    want = o.ber_sim(ebn0, 77, 12345, frames, mi, rule, llr_mode, **kw)
    llr, cw = g.channel(ebn0, 77, 12345, frames, llr_mode=llr_mode)
    got = g.ber_count(llr, cw, mi, rule, algorithm=alg).cpu().numpy()
    assert list(got) == list(want), dict(zip(oracle.COUNT_NAMES, zip(got, want)))
    got2 = g.ber_sim(ebn0, 77, 12345, frames, mi, rule, llr_mode, algorithm=alg).cpu().numpy()
    assert list(got2) == list(want)


def test_ber_sim_fused_equals_split():
    """CBP_BER_SPLIT=0 (one fused kernel) and the default split path give the same counters, with
    chunks small enough (CBP_BER_CHUNK) that the split runs several channel + decode pairs and a
    ragged last chunk; both equal the oracle's counters."""
    _need_gpu()
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, '.'); import inputs, paper_2305_05286_b200 as cbp; "
            "b, Z = inputs.config_base('C3a'); g = cbp.Code(b, Z); "
            "print(g.ber_sim(2.0, 5, 999, 2500, 30, llr_mode=1).cpu().tolist())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({"CBP_BER_SPLIT": "0"}, {"CBP_BER_SPLIT": "1", "CBP_BER_CHUNK": "1000"}):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env), capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs
    base, Z = inputs.config_base("C3a")
    want = oracle.OracleCode(base, Z).ber_sim(2.0, 5, 999, 2500, 30, llr_mode=1)
    assert outs[0] == str([int(x) for x in want])


def test_ber_count_error_paths(auto_codes):
    import ctypes
    L = cbp.lib()
    g, _ = auto_codes("C2")
    dev = torch.device("cuda", 0)
    llr, cw = g.channel(2.0, 1, 0, 4)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    ok = cbp.cbp._Opts(30, 0, 0, 0.75)

    def bc(p=None, ld=648, c=cw.data_ptr(), lw=21, frames=4, opts=ok, n=cnt.data_ptr()):
        return L.cbp_ber_count(g.handle, llr.data_ptr() if p is None else p, ld, c, lw, frames, ctypes.byref(opts), n,
                               None)
    assert bc() == 0 and int(cnt[0]) == 4
    cnt.zero_()
    assert bc(ld=640) == 1 and bc(ld=650) == 1                 # ld < N, ld % 4
    assert bc(p=llr.data_ptr() + 4) == 1                      # misaligned
    assert bc(c=None) == 1 and bc(n=None) == 1 and bc(lw=20) == 1 and bc(frames=-1) == 1
    assert bc(opts=cbp.cbp._Opts(0, 0, 0, 0.75)) == 1
    assert bc(frames=0, c=None) == 0                          # empty batch: no-op
    assert int(cnt.sum()) == 0
    g1, _ = auto_codes("C1")                                   # Z = 8: not on the one-frame-per-warp kernel
    l1, c1 = g1.channel(2.0, 1, 0, 4)
    with pytest.raises(cbp.CbpError, match="status 2"):
        g1.ber_count(l1, c1, 20)
