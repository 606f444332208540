"""GPU parity on the paper's own code families (rate-1/2 PEG codes,
N = 2048 regular (3,6) and N = 8192 irregular, max 200 iterations; QC-PEG ensemble
members from inputs/peg.py) and for the all-zero-codeword channel (CBP_TX_ZERO,
reading R23) they are simulated with.  Same bar as tests/test_gpu_parity.py:
bits, iterations, flags, edge visits and counters bit-exact."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

cbp = pytest.importorskip("paper_2305_05286_b200")

from tests.test_gpu_parity import assert_same, gpu_decode, make_code  # noqa: E402


@pytest.fixture(scope="module", params=[1, 2], ids=["P1", "P2"])
def fpl(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return request.param


@pytest.fixture(scope="module")
def codes(fpl):
    cache = {}

    def get(name):
        if name not in cache:
            base, Z = inputs.config_base(name)
            cache[name] = (make_code(base, Z, fpl), oracle.OracleCode(base, Z))
        return cache[name]
    return get


@pytest.mark.parametrize("name", ["C2", "P2048", "P8192"])
@pytest.mark.parametrize("llr_mode", [2, 3])
def test_channel_tx_zero_equals_oracle(codes, name, llr_mode):
    g, o = codes(name)
    F = 64
    llr, cw = g.channel(1.0, 11, 1000, F, llr_mode=llr_mode)
    lo, co = o.channel(1.0, 11, 1000, F, llr_mode=llr_mode)
    assert (cw.cpu().numpy() == 0).all() and (co == 0).all()
    assert (llr.cpu().numpy()[:, :o.N].view(np.uint32) == lo.view(np.uint32)).all()


def test_peg_codes_need_tx_zero(codes):
    g, _ = codes("P2048")
    with pytest.raises(cbp.CbpError, match="UNSUPPORTED|encoder"):
        g.ber_sim(2.0, 1, 0, 10, 200)
    with pytest.raises(cbp.CbpError, match="UNSUPPORTED|encoder"):
        g.channel(2.0, 1, 0, 10)
    with pytest.raises(cbp.CbpError, match="llr_mode"):
        g.ber_sim(2.0, 1, 0, 10, 200, llr_mode=4)


@pytest.mark.parametrize("name,ebn0,frames", [("P2048", 1.25, 300), ("P2048", 2.0, 400),
                                              ("P8192", 1.0, 60), ("P8192", 1.5, 80)])
def test_decode_parity_peg(codes, name, ebn0, frames):
    g, o = codes(name)
    mi = inputs.get_config(name).max_iter
    llr, _ = o.channel(ebn0, 5, 0, frames, llr_mode=oracle.TX_ZERO)
    oo = o.decode(llr, mi, want_omega=True)
    assert_same(gpu_decode(g, llr, mi), oo, o.N)
    assert (oo["iters"] > 3).mean() > 0.5            # the workload is not trivial


@pytest.mark.parametrize("alg,rule", [(0, 0), (1, 0), (0, 2), (2, 2), (3, 2)])
def test_ber_sim_tx_zero_peg_equals_oracle(codes, alg, rule):
    """Fused channel + decode + counting on P2048 (1.5 dB, near the waterfall):
    CBP log-tanh / min-sum under the belief rule and the syndrome rule, layered and
    flooding BP; counters equal the oracle's."""
    g, o = codes("P2048")
    arith = {0: oracle.FP32_CONTRACT, 1: oracle.MINSUM, 2: oracle.LBP, 3: oracle.FBP}[alg]
    F = 400 if alg != 3 else 200
    c = g.ber_sim(1.5, 21, 5000, F, 200, rule, llr_mode=2, algorithm=alg).cpu().numpy()
    co = o.ber_sim(1.5, 21, 5000, F, 200, rule, llr_mode=oracle.TX_ZERO, arith=arith)
    assert (c == co).all(), (c, co)
    assert c[2] > 0 or c[4] > 5 * F                    # errors or real iteration work


@pytest.mark.parametrize("name,ebn0,F,llr_mode", [("P8192", 1.25, 60, 2), ("C2", 1.5, 800, 2), ("C2", 1.5, 800, 3)])
def test_ber_sim_tx_zero_equals_oracle(codes, name, ebn0, F, llr_mode):
    g, o = codes(name)
    mi = inputs.get_config(name).max_iter
    c = g.ber_sim(ebn0, 4, 123, F, mi, llr_mode=llr_mode).cpu().numpy()
    co = o.ber_sim(ebn0, 4, 123, F, mi, llr_mode=llr_mode)
    assert (c == co).all(), (c, co)


@pytest.mark.parametrize("alg", [0, 1])
def test_codeword_symmetry_full_size(codes, alg):
    """Property behind R23 at the bench's size (C2, 2x10^5 frames, 2 dB): decoding the
    all-zero-codeword LLRs with the signs of a random codeword c flipped gives
    decode(L) xor c, the same iteration counts and flags, on every frame."""
    g, o = codes("C2")
    F = 200_000
    lz, _ = g.channel(2.0, 8, 0, F, llr_mode=2, want_cw=False)
    _, cw = g.channel(2.0, 9, 0, F, want_llr=False)
    bits = cw.view(torch.uint8).view(F, -1)
    c = torch.stack([(bits >> k) & 1 for k in range(8)], dim=2).reshape(F, -1)[:, :lz.shape[1]]
    flip = torch.zeros_like(lz)
    flip[:, :o.N] = 1.0 - 2.0 * c[:, :o.N].float()
    ld = lz.shape[1]
    flip[:, o.N:ld] = 1.0
    a = g.decode(lz, 30, algorithm=alg)
    b = g.decode(lz * flip, 30, algorithm=alg)
    torch.cuda.synchronize()
    assert torch.equal(a["iters"], b["iters"]) and torch.equal(a["flags"], b["flags"])
    assert torch.equal(a["bits"] ^ cw, b["bits"])
    assert (a["iters"] > 1).any()


def test_sweep_cli_peg_equals_oracle(tmp_path, capsys):
    """The resumable sweep CLI on a PEG code (all-zero codeword chosen automatically):
    its totals equal the oracle's ber_sim, and a rerun resumes from the checkpoint."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    from paper_2305_05286_b200 import sweep
    out = tmp_path / "p2048.jsonl"
    args = ["--config", "P2048", "--frames", "3000", "--chunk", "1000", "--ebn0", "2.0", "--out", str(out)]
    sweep.main(args)
    first = [json.loads(ln) for ln in capsys.readouterr().out.splitlines() if ln.startswith("{")]
    base, Z = inputs.config_base("P2048")
    want = oracle.OracleCode(base, Z).ber_sim(2.0, 1, 0, 3000, 200, llr_mode=oracle.TX_ZERO)
    got = first[0]
    assert [got[k] for k in cbp.COUNT_NAMES] == [int(x) for x in want]
    assert json.loads(out.read_text().splitlines()[0])["header"]["llr_mode"] == 2
    sweep.main(args)                                   # resumes: every chunk already recorded
    again = [json.loads(ln) for ln in capsys.readouterr().out.splitlines() if ln.startswith("{")]
    assert again == first and len(out.read_text().splitlines()) == 4
