"""CPU checks of the C-ABI boundary: the library builds, loads, and exports every
symbol include/queen.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "queen.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(queen_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ["queen_decode_residuals", "queen_apply_frame", "queen_project", "queen_bin_sort", "queen_rasterize",
              "queen_render_views"]:
        assert n in names


def test_library_builds_loads_and_exports_every_declared_symbol():
    from paper_2412_04469_b200 import build as B
    path = B.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    import paper_2412_04469_b200 as Q
    assert sorted(Q.EXPORTS) == _declared()
    L = Q.lib()
    assert L.queen_version().decode().startswith("libqueen")


def test_workspace_size_host_logic():
    import paper_2412_04469_b200 as Q
    L = Q.lib()
    nb = ctypes.c_size_t()
    assert L.queen_workspace_size(1024, 4, 64, 64, 10000, ctypes.byref(nb)) == 0 and nb.value > 0
    a = nb.value
    assert L.queen_workspace_size(1024, 8, 64, 64, 10000, ctypes.byref(nb)) == 0 and nb.value > a
    assert L.queen_workspace_size(1022, 4, 64, 64, 10000, ctypes.byref(nb)) == -2   # n_pad % 4
    assert L.queen_workspace_size(1024, 65, 64, 64, 10000, ctypes.byref(nb)) == -2  # > QUEEN_MAX_VIEWS
    assert L.queen_workspace_size(1024, 4, 64, 64, 1 << 30, ctypes.byref(nb)) == -2  # keys_cap >= 2^30
    assert L.queen_workspace_size(1024, 4, 64, 64, 100, None) == -1


def test_null_ctx_calls_fail_without_touching_the_device():
    import paper_2412_04469_b200 as Q
    L = Q.lib()
    assert L.queen_apply_frame(None, None, None, None) == -1
    assert L.queen_render_views(None, None, None, 1, None, None, None, None) == -1
    assert L.queen_check(None, None, None) == -1


def test_struct_layouts_match_header():
    import paper_2412_04469_b200 as Q
    assert ctypes.sizeof(Q.QueenCamera) == 96
    # offsets of every field as the C compiler lays them out (gcc on include/queen.h)
    import subprocess
    import tempfile
    fields = {"queen_packet": Q.QueenPacket, "queen_camera": Q.QueenCamera, "queen_proj": Q.QueenProj,
              "queen_bins": Q.QueenBins, "queen_gaussians": Q.QueenGaussians}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "queen.h"', "int main(void){"]
    for cname, py in fields.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        open(src, "w").write("\n".join(lines))
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", os.path.join(d, "l")])
        out = subprocess.check_output([os.path.join(d, "l")]).decode().split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            a, b, c = ln.split()
            got[(a, b)] = int(c)
    for cname, py in fields.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
    from harness import synth
    cam = synth.make_cameras(synth.get_config("n3dv"))[3]
    c = Q.camera_struct(cam)
    raw = np.frombuffer(bytes(c), np.float32)
    assert np.array_equal(raw[:22], cam.as_floats()[:22])


def test_wire_packet_roundtrip():
    from harness import synth
    from paper_2412_04469_b200 import packet as wire
    cfg = synth.get_config("n3dv")
    sc = synth.make_scene(cfg, n=5000)
    pkt = synth.make_packet(sc, 4)
    buf = wire.pack(pkt, frame=4, k_cap=pkt.k + 7)
    h = wire.header(buf)
    assert h["k"] == pkt.k and h["k_cap"] == pkt.k + 7 and h["lat"] == tuple(pkt.lat) and h["frame"] == 4
    lat = buf[h["lat_off"]:h["lat_off"] + sum(pkt.lat) * pkt.n_pad].view(np.int8).reshape(sum(pkt.lat), pkt.n_pad)
    assert np.array_equal(lat, pkt.latents)
    idx = buf[h["idx_off"]:h["idx_off"] + 4 * pkt.k].view(np.uint32)
    assert np.array_equal(idx, pkt.coo_idx)
    val = buf[h["val_off"]:h["val_off"] + 12 * h["k_cap"]].view(np.float32).reshape(3, h["k_cap"])
    assert np.array_equal(val[:, :pkt.k], pkt.coo_val)
    dec = buf[h["dec_off"]:h["dec_off"] + 4 * h["ndec"]].view(np.float32)
    assert np.array_equal(dec, pkt.decoders)
