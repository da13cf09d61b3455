"""GPU parity of the codec kernels (K0 quantize, K4 dequantize, K2 fused,
K3 reduce) against the reference's golden vectors and the CPU oracle.

Bar: codes and scales bit-exact; every dequantized / reduced element equal to
the reference's f64 value rounded once to the output dtype (bit-exact for
f64)."""

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle import zpp_oracle as O

pytestmark = pytest.mark.gpu

Q, M = gu.load("quant")


def _zpp():
    import paper_2306_10209_b200 as zpp
    return zpp


@pytest.mark.parametrize("case", range(len(M)))
def test_quantize_golden(case):
    zpp = _zpp()
    m = M[case]
    x = gu.to_torch(Q[f"{case}_input"], m["dtype"])
    cfg = zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"], mode=m["mode"])
    q = zpp.quantize(x, cfg)
    assert q.config.block_size == m["eff_block"]
    assert np.array_equal(q.codes.cpu().numpy(), Q[f"{case}_codes"]), m["name"]
    assert np.array_equal(q.scales.cpu().numpy(), Q[f"{case}_scales"]), m["name"]
    assert (q.payload_bytes, q.metadata_bytes, q.padding_bytes, q.wire_bytes) == (
        m["payload"], m["metadata"], m["padding"], m["wire"])
    ref = Q[f"{case}_deq"]
    for dt, name in [(torch.float64, "f64"), (torch.float32, "fp32"), (torch.float16, "fp16"),
                     (torch.bfloat16, "bf16")]:
        got = zpp.dequantize(q, dt).values.to(torch.float64).cpu().numpy()
        want = gu.round_to(ref, name)
        assert np.array_equal(got, want), (m["name"], name)


def test_known_answers():
    zpp = _zpp()
    q = zpp.quantize(torch.tensor([1.0, -1.0, 0.5, -0.5], dtype=torch.float64, device="cuda"),
                     zpp.QuantConfig(bit_width=8, block_size=8))
    assert q.scales.cpu().tolist() == [1.0 / 127.0]
    assert q.codes.cpu().numpy().view(np.int8)[:4].tolist() == [127, -127, 64, -64]
    back = zpp.dequantize(q).values.cpu().numpy()
    assert back[2] == np.float64(64) / np.float64(127)
    q = zpp.quantize(torch.zeros(16, device="cuda"), zpp.QuantConfig(bit_width=4, block_size=8))
    assert q.scales.cpu().tolist() == [0.0, 0.0] and not q.codes.any()


def test_errors_map_to_reference_exceptions():
    zpp = _zpp()
    for bad in (float("nan"), float("inf"), -float("inf")):
        for dt in (torch.float32, torch.float16, torch.bfloat16, torch.float64):
            x = torch.ones(3000, dtype=dt, device="cuda")
            x[1234] = bad
            with pytest.raises(zpp.ValidationError):
                zpp.quantize(x, zpp.QuantConfig(bit_width=8, block_size=2048))
            with pytest.raises(zpp.ValidationError):
                zpp.quantize(x, zpp.QuantConfig(bit_width=4, block_size=24))
    q = zpp.quantize(torch.ones(8, device="cuda"), zpp.QuantConfig(bit_width=8, block_size=8))
    q.codes[0] = 0x80
    with pytest.raises(zpp.IntegrityError):
        zpp.dequantize(q)
    q4 = zpp.quantize(torch.ones(8, device="cuda"), zpp.QuantConfig(bit_width=4, block_size=8))
    q4.codes[0] = 0x88
    with pytest.raises(zpp.IntegrityError):
        zpp.dequantize(q4)
    a = zpp.quantize(torch.ones(8, device="cuda"), zpp.QuantConfig(bit_width=8, block_size=8))
    b = zpp.quantize(torch.ones(16, device="cuda"), zpp.QuantConfig(bit_width=8, block_size=8))
    with pytest.raises(zpp.ValidationError):
        zpp.fused_dequant_reduce_quant([a, b], zpp.QuantConfig(bit_width=8, block_size=8))
    with pytest.raises(zpp.ValidationError):
        zpp.fused_dequant_reduce_quant([], zpp.QuantConfig(bit_width=8, block_size=8))


def test_fused_golden():
    zpp = _zpp()
    z, meta = gu.load("fused")
    for m in meta:
        i = m["idx"]
        icfg = zpp.QuantConfig(bit_width=m["in_bits"], block_size=m["in_block"])
        ocfg = zpp.QuantConfig(bit_width=m["out_bits"], block_size=m["out_block"])
        qs = [zpp.quantize(torch.from_numpy(z[f"{i}_in{j}_values"]).cuda(), icfg) for j in range(m["k"])]
        for j, q in enumerate(qs):
            assert np.array_equal(q.codes.cpu().numpy(), z[f"{i}_in{j}_codes"])
        f = zpp.fused_dequant_reduce_quant(qs, ocfg)
        assert np.array_equal(f.codes.cpu().numpy(), z[f"{i}_codes"]), m
        assert np.array_equal(f.scales.cpu().numpy(), z[f"{i}_scales"]), m
        # fused == unfused composition on the device too
        acc = zpp.dequant_reduce(qs)
        u = zpp.quantize(acc, ocfg)
        assert torch.equal(u.codes, f.codes) and torch.equal(u.scales, f.scales)


def test_fused_fp32_inputs_all_register_blocks():
    """K2 register path for every supported output block, fp32-sourced inputs."""
    zpp = _zpp()
    g = torch.Generator(device="cpu").manual_seed(5)
    for ob in (64, 128, 256, 512, 1024, 2048, 24):
        for ib in (8, 64, 512):
            for ibits, obits in ((4, 4), (8, 4), (4, 8), (8, 8)):
                n = 4 * 1024 + 512
                vals = [torch.randn(n, generator=g) * float(k + 1) for k in range(3)]
                icfg = zpp.QuantConfig(bit_width=ibits, block_size=ib)
                ocfg = zpp.QuantConfig(bit_width=obits, block_size=ob)
                qs = [zpp.quantize(v.float().cuda(), icfg) for v in vals]
                f = zpp.fused_dequant_reduce_quant(qs, ocfg)
                ins = []
                for v in vals:
                    c, s, _ = O.quantize(v.double().numpy(), ibits, ib)
                    ins.append((c, s, n, ibits, ib))
                c, s, _ = O.fused_dequant_reduce_quant(ins, obits, ob)
                assert np.array_equal(f.codes.cpu().numpy(), c), (ob, ib, ibits, obits)
                assert np.array_equal(f.scales.cpu().numpy(), s), (ob, ib, ibits, obits)


@pytest.mark.parametrize("dtype", ["fp16", "bf16", "fp32"])
@pytest.mark.parametrize("bits,block", [(8, 2048), (4, 512), (8, 64), (4, 128), (8, 256), (4, 1024), (8, 40),
                                        (4, 8), (8, 4096)])
def test_register_and_generic_paths_vs_oracle(dtype, bits, block):
    """Random heavy-tailed inputs with ragged tails through every dispatch path."""
    zpp = _zpp()
    rng = np.random.default_rng(bits * 7919 + block)
    n = 37 * block + 13
    v = np.clip(rng.normal(size=n) * np.exp(rng.normal(size=n) * 2), -60000, 60000)
    if dtype == "fp16":
        arr = v.astype(np.float16)
    elif dtype == "bf16":
        arr = (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)  # truncation is fine for inputs
    else:
        arr = v.astype(np.float32)
    x = gu.to_torch(arr, dtype)
    q = zpp.quantize(x, zpp.QuantConfig(bit_width=bits, block_size=block))
    c, s, _ = O.quantize(gu.as_f64(arr, dtype), bits, block)
    assert np.array_equal(q.codes.cpu().numpy(), c)
    assert np.array_equal(q.scales.cpu().numpy(), s)
    ref = O.dequantize(c, s, n, bits, block)
    for dt, name in [(torch.float16, "fp16"), (torch.float32, "fp32")]:
        got = zpp.dequantize(q, dt).values.to(torch.float64).cpu().numpy()
        assert np.array_equal(got, gu.round_to(ref, name))


def test_near_tie_adversarial_fp32():
    """Values engineered to land within a few ulps of k + 0.5 after scaling:
    the fp32 fast path must hand all of them to the exact f64 path."""
    zpp = _zpp()
    rng = np.random.default_rng(77)
    blocks = []
    for _ in range(512):
        m = np.float32(np.exp(rng.normal() * 10))
        k = rng.integers(-127, 127, size=2047) + 0.5
        t = (k * np.float64(m) / 127.0).astype(np.float32)
        t = np.nextafter(t, np.where(rng.random(2047) < 0.5, -np.inf, np.inf).astype(np.float32)) \
            if rng.random() < 0.5 else t
        blk = np.concatenate([[m], np.clip(t, -m, m)]).astype(np.float32)
        blocks.append(rng.permutation(blk))
    arr = np.concatenate(blocks).astype(np.float32)
    for bits in (8, 4):
        q = zpp.quantize(torch.from_numpy(arr).cuda(), zpp.QuantConfig(bit_width=bits, block_size=2048))
        c, s, _ = O.quantize(arr.astype(np.float64), bits, 2048)
        assert np.array_equal(q.codes.cpu().numpy(), c)
        assert np.array_equal(q.scales.cpu().numpy(), s)


def test_div_by_qmax_exhaustive_fp32():
    """The FMA-corrected division by qmax equals IEEE f64 division for every
    positive finite fp32 absmax (2^31 values) -- scales are bit-exact."""
    zpp = _zpp()
    lib = zpp._lib.load()
    step = 1 << 27
    out = torch.empty(step, dtype=torch.float64, device="cuda")
    for start in range(0, 0x7F800000, step):
        cnt = min(step, 0x7F800000 - start)
        bits = torch.arange(start, start + cnt, dtype=torch.int64, device="cuda").to(torch.int32)
        m = bits.view(torch.float32)
        for b, qm in ((8, 127.0), (4, 7.0)):
            zpp._lib.check(lib.zpp_scales(m.data_ptr(), zpp._lib.F32, cnt, b, out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
            md = m.double()
            # tensor / tensor: torch turns `tensor / python_scalar` into a
            # reciprocal multiply, which is not IEEE division
            want = md / torch.full_like(md, qm)
            assert torch.equal(out[:cnt], want), (start, b)


def test_div_by_qmax_random_f64():
    zpp = _zpp()
    lib = zpp._lib.load()
    g = torch.Generator(device="cuda").manual_seed(3)
    for _ in range(8):
        bits = torch.randint(0, 0x7FEFFFFFFFFFFFFF, (1 << 26,), generator=g, device="cuda", dtype=torch.int64)
        m = bits.view(torch.float64)
        out = torch.empty_like(m)
        for b, qm in ((8, 127.0), (4, 7.0)):
            zpp._lib.check(lib.zpp_scales(m.data_ptr(), zpp._lib.F64, m.numel(), b, out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
            assert torch.equal(out, m / torch.full_like(m, qm))


def test_config1_full_size_roundtrip():
    """BASELINE config 1: 16M fp32, INT8/2048, bit-exact vs the oracle at full size."""
    zpp = _zpp()
    g = torch.Generator(device="cpu").manual_seed(0)
    x = (torch.randn(1 << 24, generator=g, dtype=torch.float64) *
         torch.exp(torch.randn(1 << 24, generator=g, dtype=torch.float64))).float()
    q = zpp.quantize(x.cuda(), zpp.QuantConfig(bit_width=8, block_size=2048))
    c, s, _ = O.quantize(x.double().numpy(), 8, 2048)
    assert np.array_equal(q.codes.cpu().numpy(), c)
    assert np.array_equal(q.scales.cpu().numpy(), s)
    back = zpp.dequantize(q, torch.float32).values.cpu().numpy()
    assert np.array_equal(back, O.dequantize(c, s, x.numel(), 8, 2048).astype(np.float32))


def test_empty_and_tiny():
    zpp = _zpp()
    q = zpp.quantize(torch.zeros(0, device="cuda"), zpp.QuantConfig(bit_width=8))
    assert q.n_blocks == 0 and q.codes.numel() == 0
    assert zpp.dequantize(q).values.numel() == 0
    for n in range(1, 20):
        x = torch.linspace(-1, 1, n, device="cuda", dtype=torch.float32)
        q = zpp.quantize(x, zpp.QuantConfig(bit_width=4, block_size=8))
        c, s, _ = O.quantize(x.double().cpu().numpy(), 4, 8)
        assert np.array_equal(q.codes.cpu().numpy(), c)


def test_misaligned_input_uses_generic_path():
    zpp = _zpp()
    base = torch.randn(4096 + 3, device="cuda", dtype=torch.float16)
    x = base[3:]  # 6-byte offset: not 16-byte aligned
    q = zpp.quantize(x, zpp.QuantConfig(bit_width=8, block_size=2048))
    c, s, _ = O.quantize(x.double().cpu().numpy(), 8, 2048)
    assert np.array_equal(q.codes.cpu().numpy(), c)
    assert np.array_equal(q.scales.cpu().numpy(), s)


def test_slice_blocks_matches_direct():
    zpp = _zpp()
    vals = torch.randn(64, dtype=torch.float64, device="cuda")
    q = zpp.quantize(vals, zpp.QuantConfig(bit_width=4, block_size=16))
    part = q.slice_blocks(16, 32)
    direct = zpp.quantize(vals[16:48], zpp.QuantConfig(bit_width=4, block_size=16))
    assert torch.equal(part.codes, direct.codes) and torch.equal(part.scales, direct.scales)
    with pytest.raises(zpp.ValidationError):
        q.slice_blocks(8, 16)


def test_error_bound_half_scale():
    zpp = _zpp()
    for bits in (4, 8):
        x = torch.randn(20000, dtype=torch.float64, device="cuda") * 10
        st = zpp.quant_error_stats(x, zpp.QuantConfig(bit_width=bits, block_size=512))
        assert st.per_block_bound_violations == 0 and st.max_abs_error > 0


@pytest.mark.parametrize("src", ["fp16", "bf16", "fp32"])
@pytest.mark.parametrize("bits,block", [(8, 2048), (4, 512), (8, 64)])
def test_dequant16_fast_path_bit_exact_stress(src, bits, block):
    """4M heavy-tailed values per case through the 16-bit-output kernels
    (scale-bit-width proof path for fp16/bf16 sources, checked path for fp32
    sources): every fp16 / bf16 output equals the reference's f64 rounded once."""
    zpp = _zpp()
    rng = np.random.default_rng(hash((src, bits, block)) % 2**32)
    n = 1 << 22
    v = np.clip(rng.normal(size=n) * np.exp(rng.normal(size=n) * 3), -6e4, 6e4)
    if src == "fp16":
        arr = v.astype(np.float16)
    elif src == "bf16":
        arr = (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    else:
        arr = v.astype(np.float32)
    q = zpp.quantize(gu.to_torch(arr, src), zpp.QuantConfig(bit_width=bits, block_size=block))
    c, s, _ = O.quantize(gu.as_f64(arr, src), bits, block)
    assert np.array_equal(q.codes.cpu().numpy(), c)
    ref = O.dequantize(c, s, n, bits, block)
    for dt, name in [(torch.float16, "fp16"), (torch.bfloat16, "bf16")]:
        got = zpp.dequantize(q, dt).values.to(torch.float64).cpu().numpy()
        want = gu.round_to(ref, name)
        bad = np.flatnonzero(~((got == want) | (np.isnan(got) & np.isnan(want))))
        assert bad.size == 0, (name, bad[:5], got[bad[:5]], want[bad[:5]])


def test_wire_format_roundtrip_golden():
    """to_bytes / from_bytes (zs/quantizer.py:121-149): our bytes equal the
    reference's, and decoding them gives the reference's values."""
    zpp = _zpp()
    z, meta = gu.load("wire")
    for m in meta:
        i = m["idx"]
        cfg = zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"])
        raw = bytes(z[f"{i}_raw"].tobytes())
        back = zpp.QuantizedTensor.from_bytes(raw)
        assert back.original_len == m["n"] and back.config == cfg
        assert np.array_equal(back.codes.cpu().numpy(), z[f"{i}_codes"])
        assert np.array_equal(zpp.dequantize(back).values.cpu().numpy(), z[f"{i}_deq_from_bytes"])
        assert back.to_bytes() == raw
    with pytest.raises(zpp.IntegrityError):
        zpp.QuantizedTensor.from_bytes(b"\x00\x01")
    with pytest.raises(zpp.IntegrityError):
        zpp.QuantizedTensor.from_bytes(raw[:-1])


def test_serialization_is_deterministic():
    zpp = _zpp()
    x = torch.from_numpy(np.random.default_rng(5).normal(size=777)).cuda()
    cfg = zpp.QuantConfig(bit_width=4, block_size=64)
    assert zpp.quantize(x, cfg).to_bytes() == zpp.quantize(x, cfg).to_bytes()


def _bf16_from_f64(v):
    return gu.round_to(np.asarray(v, np.float64), "bf16")


@pytest.mark.parametrize("bits", [4, 8])
def test_exact_ties_bf16(bits):
    """bf16 blocks whose elements sit EXACTLY on a half-integer after scaling
    (x * 2*qmax / absmax odd): the reference's f64 rint goes to even.  These
    are the common case for bf16/INT4 and all of them take the f64 fix-up."""
    zpp = _zpp()
    qmax = 2 ** (bits - 1) - 1
    rng = np.random.default_rng(11 + bits)
    blocks = []
    while len(blocks) < 256:
        m = float(_bf16_from_f64(np.exp(rng.normal() * 4)))
        cand = _bf16_from_f64(rng.uniform(-m, m, size=8192))
        t = cand.astype(np.float64) * (2 * qmax) / m
        ties = cand[(np.abs(t - np.rint(t)) == 0) & (np.rint(t) % 2 == 1)]
        if len(ties) < 16:
            continue
        blk = np.resize(ties, 511)
        blocks.append(rng.permutation(np.concatenate([[m], blk])))
    arr = np.concatenate(blocks)
    x = torch.from_numpy(arr).to(torch.bfloat16).cuda()  # exact: every value is a bf16
    q = zpp.quantize(x, zpp.QuantConfig(bit_width=bits, block_size=512))
    c, s, _ = O.quantize(arr.astype(np.float64), bits, 512)
    assert np.array_equal(q.codes.cpu().numpy(), c)
    assert np.array_equal(q.scales.cpu().numpy(), s)


@pytest.mark.parametrize("n_src", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("bits,block,n", [(4, 512, 8192 + 512), (8, 2048, 3 * 2048 + 16), (8, 40, 999),
                                          (4, 24, 1000)])
def test_dequant_reduce_many_sources(n_src, bits, block, n):
    """K3 (BlockCodec.reduce_final, zs/collectives.py:71-75): f64 fold in
    source order from +0.0, for source counts around the 4-wide load batch,
    fast (16-element) and general (odd block / length) paths; f64 output
    bit-exact, fp32/fp16/bf16 outputs = the f64 result rounded once."""
    zpp = _zpp()
    rng = np.random.default_rng(n_src * 100 + bits)
    cfg = zpp.QuantConfig(bit_width=bits, block_size=block)
    vals = [rng.normal(size=n) * 10.0 ** rng.integers(-3, 3) for _ in range(n_src)]
    qs = [zpp.quantize(torch.from_numpy(v).cuda(), cfg) for v in vals]
    acc = np.zeros(n)
    for v in vals:
        c, s, _ = O.quantize(v, bits, block)
        acc = acc + O.dequantize(c, s, n, bits, block)
    assert np.array_equal(zpp.dequant_reduce(qs).cpu().numpy(), acc)
    for dt in ("fp32", "fp16", "bf16"):
        got = zpp.dequant_reduce(qs, getattr(torch, {"fp32": "float32", "fp16": "float16", "bf16": "bfloat16"}[dt]))
        assert np.array_equal(got.double().cpu().numpy(), gu.round_to(acc, dt)), dt


@pytest.mark.parametrize("n_src", [1, 2, 4, 8])
def test_fused_fixed_fanin_fast_path(n_src):
    """K2 fixed fan-in kernel (drq_fast_kernel: 1/2/4/8 sources, 512-element
    output blocks, power-of-two input blocks): codes and f64 scales bit-exact
    vs the oracle's fused_dequant_reduce_quant (zs/quantizer.py:241-258),
    including a partial last output block and bf16-sourced exact ties; a
    -8 / -128 code raises IntegrityError like the reference's dequantize."""
    zpp = _zpp()
    g = torch.Generator(device="cpu").manual_seed(50 + n_src)
    for n in (4096 + 512 + 48, 8192):
        for ib in (16, 64, 512, 2048):
            for ibits, obits in ((4, 4), (8, 4), (4, 8), (8, 8)):
                src_dt = torch.bfloat16 if (ib + ibits) % 3 == 0 else torch.float32
                vals = [(torch.randn(n, generator=g) * float(2 ** (k % 5 - 2))).to(src_dt) for k in range(n_src)]
                icfg = zpp.QuantConfig(bit_width=ibits, block_size=ib)
                ocfg = zpp.QuantConfig(bit_width=obits, block_size=512)
                qs = [zpp.quantize(v.cuda(), icfg) for v in vals]
                f = zpp.fused_dequant_reduce_quant(qs, ocfg)
                ins = []
                for v in vals:
                    c, s, _ = O.quantize(v.double().numpy(), ibits, ib)
                    ins.append((c, s, n, ibits, ib))
                c, s, _ = O.fused_dequant_reduce_quant(ins, obits, 512)
                key = (n, ib, ibits, obits, src_dt)
                assert np.array_equal(f.codes.cpu().numpy(), c), key
                assert np.array_equal(f.scales.cpu().numpy(), s), key
    # an invalid code in the last source
    icfg = zpp.QuantConfig(bit_width=4, block_size=512)
    qs = [zpp.quantize(torch.randn(4096).cuda(), icfg) for _ in range(n_src)]
    qs[-1].codes[100] = 0x88  # two -8 nibbles
    with pytest.raises(zpp.IntegrityError):
        zpp.fused_dequant_reduce_quant(qs, zpp.QuantConfig(bit_width=4, block_size=512))


@pytest.mark.parametrize("n_src", [1, 2, 4, 8])
@pytest.mark.parametrize("case", ["cancel", "near_cancel", "spread", "tiny", "huge", "ties", "zeros"])
def test_fused_int4_estimate_adversarial(n_src, case):
    """K2 INT4 -> INT4/512 goes through a certified fp32 estimate
    (drq_est_kernel) with exact f64 redo of absmax candidates and near ties:
    the cases that stress the certificate -- exact and near cancellation
    between sources (every element a redo), scales 2^40 apart, scales below
    2^-100 and above 2^100 (the exact path for the whole block), exact ties
    in the requantization, all-zero blocks -- still give the reference's codes
    and f64 scales bit for bit (zs/quantizer.py:241-258)."""
    zpp = _zpp()
    rng = np.random.default_rng(n_src * 100 + ["cancel", "near_cancel", "spread", "tiny", "huge", "ties",
                                                "zeros"].index(case))
    n = 8 * 512 + 256
    cfg = zpp.QuantConfig(bit_width=4, block_size=512)
    base = rng.normal(size=n)
    vals = []
    for k in range(n_src):
        if case == "cancel":
            v = base * (1 if k % 2 == 0 else -1)
        elif case == "near_cancel":
            v = base * (1 if k % 2 == 0 else -1) + rng.normal(size=n) * 1e-3
        elif case == "spread":
            v = rng.normal(size=n) * 2.0 ** (40 * (k % 2) - 20)
        elif case == "tiny":
            v = rng.normal(size=n) * 1e-33
        elif case == "huge":
            v = rng.normal(size=n) * 1e33
        elif case == "ties":
            v = rng.integers(-7, 8, size=n).astype(np.float64) * 0.5  # lattice values: exact ties after the fold
        else:
            v = np.zeros(n)
            v[:512] = rng.normal(size=512) if k == 0 else 0.0
        vals.append(v.astype(np.float32).astype(np.float64))
    qs = [zpp.quantize(torch.from_numpy(v).float().cuda(), cfg) for v in vals]
    f = zpp.fused_dequant_reduce_quant(qs, cfg)
    ins = []
    for v in vals:
        c, sc, _ = O.quantize(v, 4, 512)
        ins.append((c, sc, n, 4, 512))
    c, sc, _ = O.fused_dequant_reduce_quant(ins, 4, 512)
    assert np.array_equal(f.codes.cpu().numpy(), c), case
    assert np.array_equal(f.scales.cpu().numpy().view(np.uint64), np.asarray(sc).view(np.uint64)), case


def test_fused_int4_estimate_kernel_opt_in():
    """The same adversarial cases, the fixed fan-in cases and the golden K2
    cases through the opt-in certified-estimate K2 (ZPP_K2=est)."""
    import os
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", os.path.abspath(__file__),
                        "-k", "int4_estimate_adversarial or fused_fixed_fanin or fused_golden"],
                       env={**os.environ, "ZPP_K2": "est"}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("bits,block", [(8, 64), (4, 32), (8, 2048)])
def test_to_bytes_device_pack_matches_reference_layout(bits, block):
    """zpp_wire_pack (to_bytes on the device) == the reference's layout built
    on the host: '<QBI' header, numpy float16 of the f64 scales (RN-even,
    fp16 subnormals and overflow to inf included), codes with padding
    (zs/quantizer.py:121-131); from_bytes on the device inverts it."""
    import struct

    zpp = _zpp()
    rng = np.random.default_rng(bits * 1000 + block)
    n = 40 * block + block // 2 + 8
    mags = 10.0 ** rng.uniform(-9, 7, size=(n + block - 1) // block)  # scales spanning fp16's range
    x = rng.normal(size=n) * np.repeat(mags, block)[:n]
    q = zpp.quantize(torch.from_numpy(x).cuda(), zpp.QuantConfig(bit_width=bits, block_size=block))
    c, s, _ = O.quantize(x, bits, block)
    with np.errstate(over="ignore"):
        want = struct.pack("<QBI", n, bits, block) + s.astype(np.float16).tobytes() + c.tobytes()
    got = q.to_bytes()
    assert got == want
    back = zpp.QuantizedTensor.from_bytes(got)
    assert np.array_equal(back.codes.cpu().numpy(), c)
    with np.errstate(over="ignore"):
        want_abs = s.astype(np.float16).astype(np.float64) * (2 ** (bits - 1) - 1)
    assert np.array_equal(back.absmax.cpu().numpy(), want_abs)


def test_tma_fed_reduce_kernels_on_one_gpu():
    """The TMA-fed K2 / K3 (drq_tma_kernel, dr_tma_kernel) normally run only in
    multi-GPU qgZ; ZPP_FORCE_TMA=1 routes the public entry points to them so
    the fused and reduce parity tests above cover them on a single GPU too."""
    import os
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", os.path.abspath(__file__),
                        "-k", "fused_fixed_fanin or dequant_reduce_many_sources"],
                       env={**os.environ, "ZPP_FORCE_TMA": "1"}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
