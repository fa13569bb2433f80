"""C-ABI library: loads without a GPU, exports every symbol include/pf_b200.h declares, and its
host-side entry points (polygon tracing + slab index) match the oracle / reference goldens."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import port

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pf_b200.h"


@pytest.fixture(scope="module")
def native():
    from paper_2404_15217_b200 import build

    build.build()
    from paper_2404_15217_b200 import _native as N

    return N


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|void|const char\*|uint64_t)\s+(pf_\w+)\s*\(", text, re.M)))


def test_library_exports_header(native):
    syms = header_symbols()
    assert len(syms) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", str(native._LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pf_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(syms) == set(native.exported_symbols()), "python binding must cover the header exactly"
    assert native.lib().pf_abi_version() == 3


def test_errors_without_device(native):
    # argument validation runs before any CUDA call
    L = native.lib()
    rc = L.pf_read_regions(None, None, 4, 0, 0, 0, None, None, None, None)
    assert rc == native.PF_ERR_INVALID_ARG
    assert b"bad arguments" in L.pf_last_error()
    with pytest.raises(ValueError):
        native.check(rc)


def _trace(native, bits, scale, mrp):
    from paper_2404_15217_b200.foreground import BinaryMask, polygon_from_mask

    return polygon_from_mask(BinaryMask(bits, scale), min_region_px=mrp)


def test_native_trace_matches_reference(native, goldens, golden_arrays):
    poly = _trace(native, golden_arrays["blob_mask_lum"], 1 / 8, 64)
    want = goldens["blob_poly"]["rings"]
    assert len(poly.rings) == len(want)
    for a, b in zip(poly.rings, want):
        assert np.array_equal(a, np.asarray(b))
    hp = _trace(native, golden_arrays["hand_mask"], 0.5, 4)
    for a, b in zip(hp.rings, goldens["hand_poly"]["rings"]):
        assert np.array_equal(a, np.asarray(b))


def test_native_trace_random_masks_vs_oracle(native):
    rs = np.random.default_rng(7)
    for trial in range(30):
        h, w = int(rs.integers(1, 40)), int(rs.integers(1, 40))
        bits = rs.random((h, w)) < rs.uniform(0.2, 0.8)
        if trial % 3 == 0:  # smoother masks with holes
            from scipy import ndimage

            bits = ndimage.binary_opening(bits)
        scale = float(rs.choice([1.0, 0.5, 0.25, 1 / 32]))
        if not bits.any():
            from paper_2404_15217_b200.errors import EmptyForegroundError

            with pytest.raises(EmptyForegroundError):
                _trace(native, bits, scale, 1.0)
            continue
        try:
            want = port.polygon_from_mask(bits, scale, 1.0)
        except Exception:
            continue
        if not want or sum(port.shoelace(r) for r in want) <= 0:
            continue
        got = _trace(native, bits, scale, 1.0)
        assert len(got.rings) == len(want)
        for a, b in zip(got.rings, want):
            assert np.array_equal(a, b)


def test_empty_mask_raises(native):
    from paper_2404_15217_b200.errors import EmptyForegroundError

    with pytest.raises(EmptyForegroundError):
        _trace(native, np.zeros((8, 8), bool), 1.0, 64)
    with pytest.raises(EmptyForegroundError):  # only a tiny island -> filtered
        m = np.zeros((8, 8), bool)
        m[2, 2] = True
        _trace(native, m, 1.0, 64)


def test_index_blob_layout(native, goldens):
    from paper_2404_15217_b200.foreground import ForegroundPolygon

    poly = ForegroundPolygon.from_json_dict(goldens["blob_poly"])
    blob = poly.index_blob()
    hdr = np.frombuffer(blob[:32].tobytes(), dtype=np.int32)
    assert int(np.frombuffer(blob[:8].tobytes(), np.int64)[0]) == len(blob)
    n_edges, n_y = int(hdr[2]), int(hdr[3])
    assert n_edges == sum(len(r) for r in poly.rings)
    ys = np.unique(np.concatenate(poly.rings)[:, 1])
    assert n_y == len(ys)
    bbox = np.frombuffer(blob[32:64].tobytes(), np.float64)
    assert tuple(bbox) == poly.bounding_box()


def test_struct_layouts_match_header(native, tmp_path):
    """ctypes / numpy mirrors have the C header's sizes and field offsets."""
    src = tmp_path / "sizes.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "pf_b200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\","
        "sizeof(pf_slide_desc), sizeof(pf_patch_spec), sizeof(pf_sampler_config), sizeof(pf_sampler_slide),"
        "sizeof(pf_sampler_state), sizeof(pf_multicrop_config), sizeof(pf_crop_param),"
        "offsetof(pf_patch_spec, sx), offsetof(pf_sampler_state, cur_slide), offsetof(pf_crop_param, sigma));return 0;}\n"
    )
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(native.SlideDesc), native.SPEC_DTYPE.itemsize, C.sizeof(native.SamplerConfig),
            C.sizeof(native.SamplerSlide), C.sizeof(native.SamplerState), C.sizeof(native.MultiCropConfig),
            native.CROP_DTYPE.itemsize, native.SPEC_DTYPE.fields["sx"][1], native.SamplerState.cur_slide.offset,
            native.CROP_DTYPE.fields["sigma"][1]]
    assert got == want


def test_argument_validation_without_device(native):
    """Every entry point validates before touching CUDA: bad pointers / sizes fail with
    PF_ERR_INVALID_ARG and a message; empty batches are a no-op success."""
    L = native.lib()
    assert L.pf_capped_draw(1, None, None, 1, 4, None, None) == native.PF_ERR_INVALID_ARG
    assert L.pf_capped_draw(1, 8, 8, 0, 4, 8, None) == native.PF_ERR_INVALID_ARG  # empty cache
    assert b"empty cache" in L.pf_last_error()
    assert L.pf_capped_draw(1, 8, 8, 3, 0, None, None) == native.PF_OK
    assert L.pf_crop_params(0, 0, 0, -1, None, None, None) == native.PF_ERR_INVALID_ARG
    cfg = native.MultiCropConfig()
    cfg.n_global, cfg.n_local, cfg.src_size, cfg.global_size, cfg.local_size = 2, 8, 224, 224, 96
    assert L.pf_crop_params(0, 0, 0, 0, C.byref(cfg), None, None) == native.PF_OK
    assert L.pf_multicrop(None, None, None, 0, None, C.byref(cfg), 2, None, None, None, None, None) == native.PF_OK
    cfg.global_size = 100  # not a multiple of 8
    assert L.pf_multicrop(8, 8, None, 1, 8, C.byref(cfg), 2, None, None, 8, 8, None) == native.PF_ERR_INVALID_ARG
    assert L.pf_read_regions(8, 8, 0, 224, 0, 0, None, None, 8, None) == native.PF_OK
    assert L.pf_read_regions(8, 8, 1, 600, 0, 0, None, None, 8, None) == native.PF_ERR_INVALID_ARG
    assert L.pf_rrc_table_build(224, 32, 8, None) == native.PF_ERR_INVALID_ARG  # down-ratio > 3.5


def test_jpeg_record_sizes_match_host_layout(native):
    """The packed JPEG records the host preparation writes have the device structs' sizes."""
    from paper_2404_15217_b200 import store

    h, t = C.c_int32(), C.c_int32()
    assert native.lib().pf_jpeg_struct_sizes(C.byref(h), C.byref(t)) == native.PF_OK
    assert (h.value, t.value) == (store._JPEG_HUFF_BYTES, store._JPEG_TILE_BYTES)


def test_jpeg_prepare_on_host(native):
    """pf_jpeg_prepare parses Pillow's baseline files on the CPU: one Huffman/quant pool entry per
    distinct table, the 4:2:0 block list, and host fallback for progressive files."""
    import io

    import numpy as np
    from PIL import Image

    from paper_2404_15217_b200 import store

    rs = np.random.default_rng(0)
    files = []
    for prog in (False, False, True):
        buf = io.BytesIO()
        Image.fromarray(rs.integers(0, 256, (24, 40, 3), dtype=np.uint8)).save(buf, format="JPEG", quality=90,
                                                                                 progressive=prog)
        files.append(buf.getvalue())
    n = len(files)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(f) for f in files])
    data = np.frombuffer(b"".join(files), np.uint8)
    tw, th = np.full(n, 40, np.int32), np.full(n, 24, np.int32)
    dst = np.zeros(n, np.uint64)
    rec = np.zeros(n * store._JPEG_TILE_BYTES, np.uint8)
    ok = np.zeros(n, np.int32)
    pool = np.zeros(len(data) + 8, np.uint8)
    huff = np.zeros(4 * n * store._JPEG_HUFF_BYTES, np.uint8)
    quant = np.zeros(4 * n * 64, np.uint16)
    blk = [np.zeros(n * 5 * 3 * 3, np.int32) for _ in range(3)]
    px, counts = np.zeros(n, np.int64), np.zeros(7, np.int64)
    p = lambda a: a.ctypes.data  # noqa: E731
    rc = native.lib().pf_jpeg_prepare(p(data), p(off), p(tw), p(th), p(dst), n, p(rec), p(ok), p(pool), p(huff),
                                      p(quant), p(blk[0]), p(blk[1]), p(blk[2]), p(px), p(counts))
    assert rc == native.PF_OK
    assert ok.tolist() == [0, 0, 1]
    n_huff, n_quant, n_blocks = counts[:3]
    assert (n_huff, n_quant) == (4, 2)  # DC/AC x luma/chroma, shared by both baseline files
    assert n_blocks == 2 * (2 * 3 * 4 + 2 * 3 * 2)  # per file: 3x2 MCUs of 4 Y + Cb + Cr blocks
