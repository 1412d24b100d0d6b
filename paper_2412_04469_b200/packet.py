"""Frame-packet wire format (one contiguous byte buffer per frame, NCCL-broadcastable).

Carries what the paper stores per frame: the decoders D_c (fp32), the
integer latents L_c and the COO position residual (u32 indices + fp32 vectors).  Version 1
holds the latents as raw int8; version 2 (below) holds them entropy-coded as one QANS stream
per category, decoded on the GPU.  Sections are 256-B aligned.

  header: 32 x int32 little-endian
    0 magic 'QNFP'  1 version  2 frame  3 n  4 n_pad  5 sh_degree  6-10 lat_dim[5]
    11 k (live COO count; read on the device via queen_packet.k_dev)  12 k_cap
    13 dec_off 14 lat_off 15 idx_off 16 val_off 17 total_bytes 18 ndec
"""
from __future__ import annotations

import numpy as np

MAGIC = int.from_bytes(b"QNFP", "little")
VERSION = 1
HEADER_WORDS = 32
K_WORD = 11


def _al(x: int) -> int:
    return (x + 255) // 256 * 256


def category_m(deg: int):
    b = (deg + 1) ** 2
    return (4, 3, 1, 3, 3 * (b - 1))


def layout(n_pad: int, deg: int, lat, k_cap: int) -> dict:
    M = category_m(deg)
    ndec = sum(M[c] * lat[c] for c in range(5))
    SL = sum(lat)
    o = _al(HEADER_WORDS * 4)
    dec_off = o
    o = _al(o + 4 * ndec)
    lat_off = o
    o = _al(o + SL * n_pad)
    idx_off = o
    o = _al(o + 4 * k_cap)
    val_off = o
    o = _al(o + 12 * k_cap)
    return dict(ndec=ndec, SL=SL, dec_off=dec_off, lat_off=lat_off, idx_off=idx_off, val_off=val_off, total=o)


def pack(pkt, frame: int = 0, k_cap: int | None = None) -> np.ndarray:
    """Host packet (harness.synth.Packet-like: n, n_pad, deg, lat, latents int8, decoders, coo_idx, coo_val)."""
    k = int(pkt.coo_idx.shape[0])
    k_cap = k if k_cap is None else int(k_cap)
    if k > k_cap:
        raise ValueError("k > k_cap")
    L = layout(pkt.n_pad, pkt.deg, pkt.lat, k_cap)
    buf = np.zeros(L["total"], np.uint8)
    h = np.zeros(HEADER_WORDS, np.int32)
    h[0], h[1], h[2], h[3], h[4], h[5] = MAGIC, VERSION, frame, pkt.n, pkt.n_pad, pkt.deg
    h[6:11] = pkt.lat
    h[11], h[12] = k, k_cap
    h[13], h[14], h[15], h[16], h[17], h[18] = L["dec_off"], L["lat_off"], L["idx_off"], L["val_off"], L["total"], L["ndec"]
    buf[:HEADER_WORDS * 4] = h.view(np.uint8)
    buf[L["dec_off"]:L["dec_off"] + 4 * L["ndec"]] = np.ascontiguousarray(pkt.decoders, np.float32).view(np.uint8)
    buf[L["lat_off"]:L["lat_off"] + L["SL"] * pkt.n_pad] = np.ascontiguousarray(pkt.latents, np.int8).reshape(-1).view(np.uint8)
    buf[L["idx_off"]:L["idx_off"] + 4 * k] = np.ascontiguousarray(pkt.coo_idx, np.uint32).view(np.uint8)
    val = np.zeros((3, k_cap), np.float32)
    val[:, :k] = pkt.coo_val
    buf[L["val_off"]:L["val_off"] + 12 * k_cap] = val.reshape(-1).view(np.uint8)
    return buf


def header(buf: np.ndarray) -> dict:
    h = np.frombuffer(np.ascontiguousarray(buf[:HEADER_WORDS * 4]).tobytes(), np.int32)
    if int(h[0]) != MAGIC or int(h[1]) != VERSION:
        raise ValueError("bad packet magic/version")
    return dict(frame=int(h[2]), n=int(h[3]), n_pad=int(h[4]), deg=int(h[5]), lat=tuple(int(x) for x in h[6:11]),
                k=int(h[11]), k_cap=int(h[12]), dec_off=int(h[13]), lat_off=int(h[14]), idx_off=int(h[15]),
                val_off=int(h[16]), total=int(h[17]), ndec=int(h[18]))


# ---------------------------------------------------------------- version 2: entropy-coded latents
# Same header words 0-18 (lat_off unused = 0), plus:
#   19 entropy flag (1)   20-24 ans_off[5]   25-29 ans_bytes[5] (actual stream sizes; 0 if L_c = 0)
# Each category's QANS stream (csrc/entropy.cu) sits in a fixed-capacity 256-B aligned
# section (ans_cap[c]), so every frame of a stream has the same layout and the buffer can be
# NCCL-broadcast with a fixed size; only the used bytes are copied host -> device.
VERSION_ENTROPY = 2


def layout_entropy(n_pad: int, deg: int, lat, k_cap: int, ans_cap) -> dict:
    M = category_m(deg)
    ndec = sum(M[c] * lat[c] for c in range(5))
    o = _al(HEADER_WORDS * 4)
    dec_off = o
    o = _al(o + 4 * ndec)
    idx_off = o
    o = _al(o + 4 * k_cap)
    val_off = o
    o = _al(o + 12 * k_cap)
    ans_off = []
    for c in range(5):
        ans_off.append(o)
        o = _al(o + (ans_cap[c] if lat[c] else 0))
    return dict(ndec=ndec, SL=sum(lat), dec_off=dec_off, lat_off=0, idx_off=idx_off, val_off=val_off,
                ans_off=ans_off, ans_cap=list(ans_cap), total=o)


def ans_streams(pkt, encode) -> list:
    """Per-category QANS streams of a host packet's int8 latents (encode = queen_entropy_encode)."""
    out, row = [], 0
    for c in range(5):
        L = pkt.lat[c]
        out.append(encode(pkt.latents[row:row + L], pkt.n) if L else np.zeros(0, np.uint8))
        row += L
    return out


def pack_entropy(pkt, streams, frame: int = 0, k_cap: int | None = None, ans_cap=None) -> np.ndarray:
    k = int(pkt.coo_idx.shape[0])
    k_cap = k if k_cap is None else int(k_cap)
    ans_cap = [s.size for s in streams] if ans_cap is None else list(ans_cap)
    if k > k_cap or any(s.size > cap for s, cap in zip(streams, ans_cap)):
        raise ValueError("packet exceeds section capacity")
    L = layout_entropy(pkt.n_pad, pkt.deg, pkt.lat, k_cap, ans_cap)
    buf = np.zeros(L["total"], np.uint8)
    h = np.zeros(HEADER_WORDS, np.int32)
    h[0], h[1], h[2], h[3], h[4], h[5] = MAGIC, VERSION_ENTROPY, frame, pkt.n, pkt.n_pad, pkt.deg
    h[6:11] = pkt.lat
    h[11], h[12] = k, k_cap
    h[13], h[14], h[15], h[16], h[17], h[18] = L["dec_off"], 0, L["idx_off"], L["val_off"], L["total"], L["ndec"]
    h[19] = 1
    h[20:25] = L["ans_off"]
    h[25:30] = [s.size for s in streams]
    buf[:HEADER_WORDS * 4] = h.view(np.uint8)
    buf[L["dec_off"]:L["dec_off"] + 4 * L["ndec"]] = np.ascontiguousarray(pkt.decoders, np.float32).view(np.uint8)
    buf[L["idx_off"]:L["idx_off"] + 4 * k] = np.ascontiguousarray(pkt.coo_idx, np.uint32).view(np.uint8)
    val = np.zeros((3, k_cap), np.float32)
    val[:, :k] = pkt.coo_val
    buf[L["val_off"]:L["val_off"] + 12 * k_cap] = val.reshape(-1).view(np.uint8)
    for c in range(5):
        if streams[c].size:
            buf[L["ans_off"][c]:L["ans_off"][c] + streams[c].size] = streams[c]
    return buf


def header_entropy(buf: np.ndarray) -> dict:
    h = np.frombuffer(np.ascontiguousarray(buf[:HEADER_WORDS * 4]).tobytes(), np.int32)
    if int(h[0]) != MAGIC or int(h[1]) != VERSION_ENTROPY:
        raise ValueError("not an entropy-coded packet")
    d = dict(frame=int(h[2]), n=int(h[3]), n_pad=int(h[4]), deg=int(h[5]), lat=tuple(int(x) for x in h[6:11]),
             k=int(h[11]), k_cap=int(h[12]), dec_off=int(h[13]), lat_off=0, idx_off=int(h[15]), val_off=int(h[16]),
             total=int(h[17]), ndec=int(h[18]), ans_off=[int(x) for x in h[20:25]], ans_bytes=[int(x) for x in h[25:30]])
    d["used"] = max([d["val_off"] + 12 * d["k_cap"]] + [o + b for o, b in zip(d["ans_off"], d["ans_bytes"])])
    return d
