"""GPU parity: the CUDA path through the C ABI against the CPU oracle,
element by element on the same seeded inputs.  Integer work => bit-exact."""
import os
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O
import layout_decode as LD

pytestmark = pytest.mark.gpu


def _wino():
    import paper_1901_01965_b200 as W
    return W


FUSED, STAGED = 1, 2   # WINO_PATH_FUSED / WINO_PATH_STAGED (WINO_PATH_AUTO = 0)
PATHS = [pytest.param(FUSED, id="fused"), pytest.param(STAGED, id="staged")]


def _run(x, w, layout, pad=1, scaling=True, out_mode=1, M0=1, S=0, chunk_mb=None, path=FUSED):
    W = _wino()
    if chunk_mb is not None:
        os.environ["WINO_CHUNK_MB"] = str(chunk_mb)
    try:
        if layout == O.NCHW:
            n, ci, h, wd = x.shape
        else:
            n, h, wd, ci = x.shape
        co = w.shape[0]
        conv = W.WinoConv2d(n, h, wd, ci, co, pad, layout, scaling, out_mode, path=path)
    finally:
        os.environ.pop("WINO_CHUNK_MB", None)
    xd = torch.from_numpy(x).cuda(); wdv = torch.from_numpy(w).cuda()
    conv.transform_filter(wdv)
    y = conv(xd, M0, S)
    torch.cuda.synchronize()
    return conv, y.cpu().numpy()


def _check_layer(x, w, layout, pad=1, scaling=True, chunk_mb=None, intermediates=True, path=FUSED):
    conv, y32 = _run(x, w, layout, pad, scaling, 1, chunk_mb=chunk_mb, path=path)
    ref = O.wino_conv(x, w, pad, layout, scaling=scaling, want_M=intermediates)
    np.testing.assert_array_equal(y32, ref.out32)
    if not scaling:
        np.testing.assert_array_equal(y32.astype(np.int64), O.direct_conv(x, w, pad, layout))
    if intermediates:
        info = conv.info
        co, ci = w.shape[0], (w.shape[1] if layout == O.NCHW else w.shape[3])
        # K1: codes and W' operand planes, byte exact
        _, Wp, codes = O.filter_transform(w, layout, scaling=scaling)
        np.testing.assert_array_equal(conv.codes.cpu().numpy(), codes)
        wbuf = conv.w_wino.cpu().numpy()
        if path == FUSED and info.packing == 4:   # quarter-K packed W' (c_in <= 8)
            wr, wre, wim, dup_ok = LD.decode_w_qk(wbuf, info.cout_pad, ci)
            er, ere, eim = LD.complex_to_values(Wp)
            np.testing.assert_array_equal(wr[:, :co], er)
            np.testing.assert_array_equal(wre[:, :co], ere)
            np.testing.assert_array_equal(wim[:, :co], eim)
            assert dup_ok, "packed B: -Wi / Wr duplicates, zero rows and the other slot's K half"
            for a_ in (wr, wre, wim):
                assert not a_[:, co:, :].any()
        elif path == FUSED:
            wr, wre, wim, dup_ok = LD.decode_w_fused(wbuf, info.cout_pad, info.cin_pad // 32, info.cin_pad)
            er, ere, eim = LD.complex_to_values(Wp)
            np.testing.assert_array_equal(wr[:, :co, :ci], er)
            np.testing.assert_array_equal(wre[:, :co, :ci], ere)
            np.testing.assert_array_equal(wim[:, :co, :ci], eim)
            assert dup_ok, "B1 rows must hold -Wi and Wr"
            for a_ in (wr, wre, wim):
                assert not a_[:, co:, :].any() and not a_[:, :, ci:].any()
        else:
            wpl = LD.decode_w_staged(wbuf, info.cout_pad, info.n_block, info.cin_pad // 32, info.cin_pad)
            np.testing.assert_array_equal(wpl[:, :co, :ci], LD.complex_to_planes(Wp))
            assert not wpl[:, co:, :].any() and not wpl[:, :, ci:].any()
        if info.n_chunks == 1:
            # K2: V planes of every tile, byte exact
            T = int(info.tiles)
            vbuf = conv.v_image().cpu().numpy()
            D = O.input_transform(x, pad, layout)
            if path == FUSED:
                vr, vre, vim = (LD.decode_v_qk(vbuf, T, ci) if info.packing == 4 else
                                LD.decode_v_fused(vbuf, T, info.cin_pad // 32, info.cin_pad))
                er, ere, eim = LD.complex_to_values(D)
                np.testing.assert_array_equal(vr[:, :, :ci], er)
                np.testing.assert_array_equal(vre[:, :, :ci], ere)
                np.testing.assert_array_equal(vim[:, :, :ci], eim)
                return conv
            vpl = LD.decode_v(vbuf, T, info.cin_pad // 32, info.cin_pad)
            np.testing.assert_array_equal(vpl[:, :, :ci], LD.complex_to_planes(D))
            # K3: GEMMs + Karatsuba recombination + reverse scaling == oracle M''
            mraw = conv.m_raw().cpu().numpy()
            ms = LD.decode_m(mraw, T, co, info.cout_pad, info.n_block, info.chunk_tiles_pad)
            real, re, im = ms[:16], ms[16:26], ms[26:36]
            Mo = ref.Mpp.transpose(2, 0, 1, 3)      # [36][T][co][2]
            np.testing.assert_array_equal(real, Mo[LD.REAL_POS, :, :, 0])
            np.testing.assert_array_equal(re, Mo[LD.CPX_POS, :, :, 0])
            np.testing.assert_array_equal(im, Mo[LD.CPX_POS, :, :, 1])
    return conv


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
@pytest.mark.parametrize("scaling", [False, True])
def test_c1_all_stages(layout, scaling, path):
    """BASELINE configs[0]: batch 1, 8x8, 4->4, scaling off then on; every
    kernel's output (codes, W', V, M'' on the staged path, y) against the oracle."""
    x, w = synth.config_inputs("C1", layout)
    _check_layer(x, w, layout, 1, scaling, path=path)


@pytest.mark.parametrize("case", [
    # n, h, w, cin, cout, pad, layout    -- ragged maps, several tile / cout blocks, K tails
    (2, 40, 37, 17, 70, 1, O.NHWC),
    (1, 23, 30, 64, 16, 0, O.NHWC),
    (3, 13, 9, 3, 5, 1, O.NCHW),
    (1, 3, 3, 1, 1, 0, O.NHWC),
    (2, 1, 1, 2, 3, 1, O.NCHW),
    (1, 57, 11, 40, 33, 1, O.NCHW),
    (4, 18, 18, 96, 128, 1, O.NHWC),
    # the fused kernel's stage variants: 3 K steps (one 80 KB stage per slot-group), 7 K steps (two
    # 4-K-step stages, the second a tail), 10 K steps (the general ring)
    (2, 14, 10, 80, 48, 1, O.NCHW),
    (2, 11, 13, 200, 24, 1, O.NHWC),
    (1, 9, 9, 300, 20, 1, O.NHWC),
    # quarter-K packing (NHWC int8, c_in <= 8): several 128-tile blocks with a ragged last one, a cout tail
    (3, 30, 34, 3, 64, 1, O.NHWC),
    (2, 17, 22, 8, 20, 0, O.NHWC),
])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", PATHS)
def test_random_shapes_all_stages(case, scaling, path):
    n, h, wd, ci, co, pad, layout = case
    rng = np.random.default_rng(zlib.crc32(repr((case, scaling)).encode()))
    x, w = synth.random_layer(rng, n, h, wd, ci, co, layout)
    _check_layer(x, w, layout, pad, scaling, path=path)


@pytest.mark.parametrize("xv,wv", [(-128, -128), (127, 127), (-128, 127)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", PATHS)
def test_extremes(xv, wv, scaling, path):
    x = np.full((2, 12, 13, 40), xv, np.int8); w = np.full((24, 3, 3, 40), wv, np.int8)
    _check_layer(x, w, O.NHWC, 1, scaling, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_multi_chunk_matches_single_chunk(path):
    rng = np.random.default_rng(77)
    x, w = synth.random_layer(rng, 24, 20, 20, 64, 48, O.NHWC)
    conv, y = _run(x, w, O.NHWC, scaling=True, chunk_mb=1, path=path)
    assert conv.info.n_chunks > 1
    np.testing.assert_array_equal(y, O.wino_conv(x, w, 1, O.NHWC, scaling=True).out32)


@pytest.mark.parametrize("shape", [(3, 30, 34, 3, 64), (2, 17, 22, 5, 96), (1, 9, 13, 1, 32), (2, 21, 19, 8, 48)])
def test_quarter_k_paired_int8_output(shape):
    """Quarter-K packing (c_in <= 8) with int8 NHWC output: an even number of 16-cout blocks runs as cout-block
    pairs on one CTA whose outputs leave as whole 32-byte sectors (c_out 64, 96, 32); c_out 48 (three blocks)
    keeps single units.  Several tile blocks, ragged maps, requantisation with and without rounding."""
    W = _wino()
    n, h, wd, ci, co = shape
    rng = np.random.default_rng(90 + co)
    x, w = synth.random_layer(rng, n, h, wd, ci, co, O.NHWC)
    for M0, S in [(1, 0), (1, 9), (3, 11)]:
        _, y8 = _run(x, w, O.NHWC, scaling=True, out_mode=0, M0=M0, S=S, path=W.WINO_PATH_FUSED)
        np.testing.assert_array_equal(y8, O.wino_conv(x, w, 1, O.NHWC, scaling=True, M0=M0, S=S).y8)
    # several chunks on two lanes
    conv = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=W.WINO_PATH_FUSED,
                        workspace_mb=1, lanes=2)
    conv.transform_filter(torch.from_numpy(w).cuda())
    np.testing.assert_array_equal(conv(torch.from_numpy(x).cuda(), 1, 9).cpu().numpy(),
                                  O.wino_conv(x, w, 1, O.NHWC, scaling=True, M0=1, S=9).y8)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cout", [20, 32])
@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
def test_int8_requant_output(layout, cout, path):
    rng = np.random.default_rng(5)
    x, w = synth.random_layer(rng, 2, 15, 14, 24, cout, layout)
    for M0, S in [(1, 0), (1, 9), (3, 11), (7, 1), (1, 20), (1, 24), (5, 40)]:
        _, y8 = _run(x, w, layout, scaling=True, out_mode=0, M0=M0, S=S, path=path)
        ref = O.wino_conv(x, w, 1, layout, scaling=True, M0=M0, S=S)
        np.testing.assert_array_equal(y8, ref.y8)


@pytest.mark.parametrize("path", PATHS)
def test_max_cin_unscaled_896_and_scaled_768(path):
    rng = np.random.default_rng(9)
    for ci, scaling in [(896, False), (768, True)]:
        x = rng.integers(-128, 128, (1, 6, 7, ci)).astype(np.int8)
        w = np.where(rng.integers(0, 2, (3, 3, 3, ci)) == 1, 127, -128).astype(np.int8)
        _check_layer(x, w, O.NHWC, 1, scaling, intermediates=False, path=path)


def test_plan_rejects():
    W = _wino()
    L = W._lib
    bad = [dict(pad=2), dict(c_in=897, filter_scaling=0), dict(c_in=769, filter_scaling=1), dict(h=0),
           dict(h=1, pad=0), dict(filter_target_max=127, path=1)]   # 127 needs the staged path
    for kw in bad:
        d = dict(n=1, h=8, w=8, c_in=4, c_out=4, pad=1, layout=1, filter_scaling=1, filter_target_max=255,
                 out_mode=0)
        d.update(kw)
        with pytest.raises(W.WinoError) as e:
            L.wino_plan(L.wino_conv_desc(**d), 0)
        assert e.value.status == L.WINO_ERR_UNSUPPORTED
    d = L.wino_conv_desc(1, 8, 8, 4, 4, 1, 7, 1, 255, 0, 0)
    with pytest.raises(W.WinoError) as e:
        L.wino_plan(d, 0)
    assert e.value.status == L.WINO_ERR_INVALID_ARG


def test_conv_rejects_bad_requant_and_null():
    W = _wino()
    conv = W.WinoConv2d(1, 8, 8, 4, 4, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8)
    x = torch.zeros(conv.x_shape, dtype=torch.int8, device="cuda")
    with pytest.raises(W.WinoError) as e:
        conv(x, requant_mult=0, requant_shift=3)
    assert e.value.status == W._lib.WINO_ERR_RANGE
    with pytest.raises(W.WinoError):
        W._lib.wino_conv2d_int8(conv.plan, 0, conv.w_wino.data_ptr(), conv.codes.data_ptr(), 1, 0, 0,
                                conv.workspace.data_ptr(), 0)


def test_host_entry_point_matches_device_path():
    W = _wino()
    x, w = synth.config_inputs("C2", n=3)
    conv = W.WinoConv2d(3, 56, 56, 64, 64, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8)
    conv.transform_filter(torch.from_numpy(w).cuda())
    S = synth.requant_shift(synth.CONFIGS["C2"].layers[0])
    y_dev = conv(torch.from_numpy(x).cuda(), 1, S)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(conv.y_shape, dtype=torch.int8).pin_memory()
    xd = torch.empty(conv.x_shape, dtype=torch.int8, device="cuda")
    yd = torch.empty(conv.y_shape, dtype=torch.int8, device="cuda")
    conv.call_host(xh, yh, xd, yd, 1, S)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(yh.numpy(), y_dev.cpu().numpy())
    np.testing.assert_array_equal(yh.numpy(), O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=S).y8)


def test_invalid_scale_code_is_range_at_the_boundary():
    """a scale_codes entry that does not decode to n in [8, 15] (A4) is
    WINO_ERR_RANGE from wino_conv2d_int8 itself (nothing enqueued); the same buffer made valid
    passes after wino_validate_codes; codes written by wino_transform_filter are accepted."""
    W = _wino()
    L = W._lib
    for path in (FUSED, STAGED):
        conv = W.WinoConv2d(1, 8, 8, 4, 4, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=path)
        x, w = synth.config_inputs("C1", O.NHWC)
        xd = torch.from_numpy(x).cuda()
        conv.transform_filter(torch.from_numpy(w).cuda())
        good = conv(xd).cpu().numpy()                          # the plan's own codes: accepted
        np.testing.assert_array_equal(good, O.wino_conv(x, w, 1, O.NHWC, True).out32)
        bad = conv.codes.clone()
        bad[1, 3] = 5 << 2                                      # n = 5: not a code of P:330
        y = torch.full(conv.y_shape, 7, dtype=torch.int32, device="cuda")
        with pytest.raises(W.WinoError) as e:
            conv(xd, y=y, codes=bad)
        assert e.value.status == L.WINO_ERR_RANGE
        assert (y == 7).all().item()                            # nothing was enqueued
        with pytest.raises(W.WinoError) as e:
            L.wino_validate_codes(conv.plan, bad.data_ptr(), conv.workspace.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream)
        assert e.value.status == L.WINO_ERR_RANGE
        bad[1, 3] = conv.codes[1, 3]                            # repaired, re-validated, accepted
        L.wino_validate_codes(conv.plan, bad.data_ptr(), conv.workspace.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(conv(xd, codes=bad).cpu().numpy(), good)
        for v in (1, 31, 64, 200):                              # n < 8, n = 7 max, > 6 bits
            b2 = conv.codes.clone(); b2[0, 0] = v
            with pytest.raises(W.WinoError) as e:
                conv(xd, codes=b2)
            assert e.value.status == L.WINO_ERR_RANGE, v


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("lanes", [2, 3])
@pytest.mark.parametrize("shape", [(13, 30, 26, 64, 48), (13, 60, 52, 3, 48)])   # the second: quarter-K packing
def test_chunk_lanes_match_the_oracle(path, lanes, shape):
    """wino_conv_desc.lanes: chunks on concurrent streams with their own V (+ M'') buffers give the oracle's
    result, eagerly and inside a captured CUDA graph (the fork/join is captured)."""
    W = _wino()
    rng = np.random.default_rng(50 + lanes)
    n, h, wd, ci, co = shape
    x, w = synth.random_layer(rng, n, h, wd, ci, co, O.NHWC)
    conv = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=path, workspace_mb=1,
                        lanes=lanes)
    assert conv.info.n_chunks >= 2 and conv.info.lanes == min(lanes, conv.info.n_chunks)
    conv.transform_filter(torch.from_numpy(w).cuda())
    xd = torch.from_numpy(x).cuda()
    ref = O.wino_conv(x, w, 1, O.NHWC, True).out32
    np.testing.assert_array_equal(conv(xd).cpu().numpy(), ref)
    y = torch.zeros(conv.y_shape, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            conv(xd, y=y, stream=st)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("shape", [(2, 16, 24, 32, 48), (1, 14, 10, 64, 16), (3, 28, 28, 40, 64), (1, 9, 7, 8, 32)])
def test_fused_pool_output_mode(path, shape):
    """WINO_OUT_INT8_POOL2 (the VGG stack's 2x2/2 max pool fused into the output stage) equals the oracle's
    requantised output followed by its max pool, incl. odd / non-multiple-of-4 maps (floor)."""
    W = _wino()
    n, h, w_, ci, co = shape
    rng = np.random.default_rng(sum(shape))
    x, w = synth.random_layer(rng, n, h, w_, ci, co, O.NHWC)
    conv = W.WinoConv2d(n, h, w_, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8_POOL2, path=path, lanes=2,
                        workspace_mb=1)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda(), 1, 9).cpu().numpy()
    ref = O.maxpool2(O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=9).y8, O.NHWC)
    assert y.shape == ref.shape
    np.testing.assert_array_equal(y, ref)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("variant", ["i32", "i8_lanes", "pool", "f2", "u8", "qk"])
def test_kernels_write_only_inside_their_buffers(path, variant):
    """compute-sanitizer is closed on this pool, so out-of-bounds WRITES are caught with canaries: every
    device buffer the library writes (W', codes, workspace, y) sits inside a larger allocation whose 4 KB
    guard bands on both sides hold a pattern that must survive K1..K4 unchanged; the result is also the
    oracle's.  Covers a partial last tile block (3 x 30 x 34 maps), two chunks and lanes."""
    W = _wino()
    L = W._lib
    rng = np.random.default_rng(71)
    n, h, w_, ci, co = 3, 30, 34, 40, 32
    if variant == "qk":   # c_in <= 8: quarter-K packed V and W' on the fused path
        ci = 5
    x, w = synth.random_layer(rng, n, h, w_, ci, co, O.NHWC)
    kw = dict(path=path)
    out_mode = W.WINO_OUT_INT32
    if variant == "i8_lanes":
        out_mode, kw["lanes"], kw["workspace_mb"] = W.WINO_OUT_INT8, 2, 1
    elif variant == "pool":
        out_mode = W.WINO_OUT_INT8_POOL2
    elif variant == "f2":
        kw["algorithm"] = W.WINO_ALG_F2X2
    elif variant == "u8":
        kw.update(input_type=W.WINO_IN_UINT8, x_zero_point=128, w_zero_point=128)
    conv = W.WinoConv2d(n, h, w_, ci, co, 1, W.WINO_NHWC, True, out_mode, **kw)
    G = 4096
    def guarded(nbytes):
        buf = torch.full((nbytes + 2 * G,), 0x5A, dtype=torch.uint8, device="cuda")
        return buf, buf[G:G + nbytes]
    i = conv.info
    wbuf, wwin = guarded(i.filter_bytes)
    cbuf, cod = guarded(i.codes_bytes)
    sbuf, wsp = guarded(i.workspace_bytes)
    ybytes = i.y_bytes
    ybuf, yv = guarded(ybytes)
    to_in = (lambda a: (a.astype(np.int16) + 128).astype(np.uint8)) if variant == "u8" else (lambda a: a)
    xd = torch.from_numpy(np.ascontiguousarray(to_in(x))).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(to_in(w))).cuda()
    sp = torch.cuda.current_stream().cuda_stream
    L.wino_transform_filter(conv.plan, wd.data_ptr(), wwin.data_ptr(), cod.data_ptr(), sp)
    L.wino_conv2d_int8(conv.plan, xd.data_ptr(), wwin.data_ptr(), cod.data_ptr(), 1, 9, yv.data_ptr(),
                       wsp.data_ptr(), sp)
    torch.cuda.synchronize()
    for buf in (wbuf, cbuf, sbuf, ybuf):
        assert bool((buf[:G] == 0x5A).all()) and bool((buf[-G:] == 0x5A).all())
    if variant == "f2":
        ref = O.wino2_conv(x, w, 1, O.NHWC, True).out32
    elif variant == "pool":
        ref = O.maxpool2(O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=9).y8, O.NHWC)
    elif variant == "i8_lanes":
        ref = O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=9).y8
    else:
        ref = O.wino_conv(x, w, 1, O.NHWC, True).out32
    got = yv.view(torch.int32 if ref.dtype == np.int32 else torch.int8).cpu().numpy().reshape(ref.shape)
    np.testing.assert_array_equal(got, ref)


def test_check_codes_and_maxpool():
    W = _wino()
    conv = W.WinoConv2d(1, 8, 8, 4, 4, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    codes = torch.zeros((4, 36), dtype=torch.uint8, device="cuda"); codes[1, 3] = 8 << 2 | 1
    W._lib.wino_check_codes(conv.plan, codes.data_ptr(), bad.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert bad.item() == 0
    codes[2, 5] = 5 << 2
    W._lib.wino_check_codes(conv.plan, codes.data_ptr(), bad.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert bad.item() == 1
    rng = np.random.default_rng(1)
    for layout in (O.NHWC, O.NCHW):
        x = rng.integers(-128, 128, (2, 10, 12, 7)).astype(np.int8)
        if layout == O.NCHW:
            x = np.ascontiguousarray(x.transpose(0, 3, 1, 2))
        y = W.maxpool2(torch.from_numpy(x).cuda(), layout).cpu().numpy()
        np.testing.assert_array_equal(y, O.maxpool2(x, layout))
    # the vectorised NHWC path (c % 16 == 0): signed byte max over the int8 extremes, odd map sizes
    for (h, w, c) in [(10, 13, 32), (224, 224, 64), (3, 2, 16)]:
        x = rng.integers(-128, 128, (2, h, w, c)).astype(np.int8)
        x[0, 0, 0, :8] = -128
        x[0, 0, 1, 8:] = 127
        y = W.maxpool2(torch.from_numpy(x).cuda(), O.NHWC).cpu().numpy()
        np.testing.assert_array_equal(y, O.maxpool2(x, O.NHWC))


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_size_configs_every_image(name, path):
    """Full BASELINE sizes in the bench launch configuration (NHWC, int8 out,
    default chunking): EVERY image of the batch compared bit-exactly with the
    oracle run on the whole batch."""
    W = _wino()
    layer = synth.CONFIGS[name].layers[0]
    x, w = synth.config_inputs(name)
    S = synth.requant_shift(layer)
    conv = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, 1, W.WINO_NHWC, True,
                        W.WINO_OUT_INT8, path=path)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda(), 1, S).cpu().numpy()
    ref = O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=S)
    assert y.shape == ref.y8.shape
    np.testing.assert_array_equal(y, ref.y8)
    # codes computed on the device equal the oracle's
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), O.filter_transform(w, O.NHWC, True)[2])


def _oracle_stack(x, ws, shifts, pools):
    outs, cur = [], x
    for i, w in enumerate(ws):
        cur = O.wino_conv(cur, w, 1, O.NHWC, scaling=True, M0=1, S=shifts[i]).y8
        if i in pools:
            cur = O.maxpool2(cur, O.NHWC)
        outs.append(cur)
    return outs


@pytest.mark.parametrize("path", [pytest.param(STAGED, id="staged"), pytest.param(0, id="auto")])
def test_vgg16_stack_full_size_sampled(path):
    """BASELINE configs[4] at full size (13 layers, 224x224, batch 256, requantised,
    max-pooled): images 0 and 255 compared layer by layer with the oracle; all layers staged,
    and per-layer AUTO as bench.py runs it (fused for the five layers with c_in <= 128)."""
    from paper_1901_01965_b200.stack import ConvStack
    cfg = synth.CONFIGS["C5"]
    shifts = synth.stack_shifts("C5")
    x, ws = synth.stack_inputs("C5")
    st = ConvStack(x.shape[0], cfg.layers, cfg.pools_after, shifts, path=path)
    if path == 0:
        assert [c.info.path for c in st.convs] == [FUSED] * 5 + [STAGED] * 8
    wd = [torch.from_numpy(w).cuda() for w in ws]
    if path == 0:     # as bench.py runs it: filter transforms forked onto a side stream (ConvStack.step)
        st.step(torch.from_numpy(x).cuda(), wd)
    else:
        st.transform_filters(wd)
        st(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    for img in (0, x.shape[0] - 1):
        ref = _oracle_stack(x[img:img + 1], ws, shifts, set(cfg.pools_after))
        for i in range(len(ws)):
            got = (st.pooled[i] if i in st.pooled else st.outs[i])[img:img + 1].cpu().numpy()
            np.testing.assert_array_equal(got, ref[i], err_msg=f"layer {i} image {img}")
    # the activations stay informative (requant shifts neither saturate nor vanish)
    last = (st.pooled.get(len(ws) - 1, st.outs[-1])).cpu().numpy()
    assert 4 < np.abs(last.astype(np.int32)).mean() < 100


def test_auto_path_choice_and_parity():
    """WINO_PATH_AUTO resolves to fused for F(2x2) and for F(4x4) at c_in <= 128 (target 255), staged
    otherwise (info.path reports it), and either way the result is the oracle's."""
    W = _wino()
    for (ci, co, kw, want) in [(64, 64, {}, W.WINO_PATH_FUSED), (128, 128, {}, W.WINO_PATH_FUSED),
                               (128, 256, {}, W.WINO_PATH_FUSED), (256, 256, {}, W.WINO_PATH_STAGED), (129, 64, {}, W.WINO_PATH_STAGED),
                               (300, 64, {}, W.WINO_PATH_STAGED), (512, 512, {}, W.WINO_PATH_STAGED),
                               (64, 64, dict(algorithm=W.WINO_ALG_F2X2), W.WINO_PATH_FUSED),
                               (512, 64, dict(algorithm=W.WINO_ALG_F2X2), W.WINO_PATH_FUSED),
                               (64, 64, dict(input_type=W.WINO_IN_UINT8, x_zero_point=3, w_zero_point=250),
                                W.WINO_PATH_FUSED),
                               (64, 64, dict(filter_target_max=127), W.WINO_PATH_STAGED)]:
        conv = W.WinoConv2d(1, 9, 10, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_AUTO, **kw)
        assert conv.info.path == want, (ci, co, kw)
    rng = np.random.default_rng(77)
    x, w = synth.random_layer(rng, 2, 13, 11, 40, 24, O.NHWC)
    conv = W.WinoConv2d(2, 13, 11, 40, 24, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_AUTO)
    conv.transform_filter(torch.from_numpy(w).cuda())
    np.testing.assert_array_equal(conv(torch.from_numpy(x).cuda()).cpu().numpy(),
                                  O.wino_conv(x, w, 1, O.NHWC, True).out32)


@pytest.mark.gpu
def test_staged_gemm_cta_pair_variant_matches_the_oracle():
    """WINO_K3_PAIR=1 (read once per process, so in a subprocess): the staged GEMM on CTA pairs
    (tcgen05.mma.cta_group::2, M = 256, B split between the pair) -- an odd tile-block count (the last block
    unpaired), c_out 64 (n_block 64), scaling on, int32 out -- equals the oracle."""
    import subprocess, sys, textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent("""
        import sys, numpy as np, torch
        sys.path.insert(0, %r); sys.path.insert(0, %r)
        import synth, paper_1901_01965_b200 as W
        from oracle import oracle as O
        rng = np.random.default_rng(7)
        x, w = synth.random_layer(rng, 6, 28, 28, 96, 64, O.NHWC)   # 6 x 49 = 294 tiles: three blocks (one unpaired)
        c = W.WinoConv2d(6, 28, 28, 96, 64, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_STAGED)
        c.transform_filter(torch.from_numpy(w).cuda())
        y = c(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(y, O.wino_conv(x, w, 1, O.NHWC, True).out32)
        x, w = synth.random_layer(rng, 7, 30, 30, 64, 128, O.NHWC)  # 7 x 64 = 448 tiles: four blocks, two cout blocks
        c = W.WinoConv2d(7, 30, 30, 64, 128, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_STAGED)
        c.transform_filter(torch.from_numpy(w).cuda())
        y = c(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(y, O.wino_conv(x, w, 1, O.NHWC, True).out32)
        print("ok")
    """ % (root, os.path.join(root, "tests")))
    env = dict(os.environ, WINO_K3_PAIR="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
