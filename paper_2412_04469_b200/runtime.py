"""Per-frame player over libqueen: resident Gaussian SoA, A_t = A_{t-1} + R_t, multi-view render.

Everything here is argument marshalling and buffer management (torch memory,
streams); every step of the path runs in libqueen's kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import (QUEEN_LAT_F32, QUEEN_LAT_INT8, QUEEN_MAX_VIEWS, QUEEN_POS_COO, QUEEN_POS_GATES, Context,
               QueenError, camera_array, gaussians_struct, packet_struct, queen_apply_frame,
               queen_densify, queen_entropy_decode_frame, queen_render_mask, queen_render_views,
               queen_render_views_f16, queen_render_views_rgb8, queen_render_views_rgb10, queen_set_blend_stream,
               queen_wait_binned,
               queen_wait_projected)
from . import packet as wire


_OUT_FNS = {"f32": (queen_render_views, torch.float32), "rgb8": (queen_render_views_rgb8, torch.uint8),
            "f16": (queen_render_views_f16, torch.float16),
            "rgb10": (queen_render_views_rgb10, torch.int32)}


def _out_fn(rgb8, out):
    """Output format of a render call: rgb8=True or a uint8 `out` -> u8 display format; a float16
    `out` -> binary16; an int32 `out` ([V][H][W]) -> packed 10-bit R10G10B10A2; else fp32."""
    if rgb8 is True or rgb8 == "rgb8" or (out is not None and out.dtype == torch.uint8):
        fmt = "rgb8"
    elif rgb8 == "f16" or (out is not None and out.dtype == torch.float16):
        fmt = "f16"
    elif rgb8 == "rgb10" or (out is not None and out.dtype == torch.int32):
        fmt = "rgb10"
    else:
        fmt = "f32"
    fn, dt = _OUT_FNS[fmt]
    if fmt != "f32" and (out is None or out.dtype != dt):
        shape = "[V][H][W]" if fmt == "rgb10" else "[V][3][H][W]"
        raise ValueError(f"{fmt} rendering needs an out tensor of dtype {dt} {shape}")
    return fn


class DevicePacket:
    """A frame packet resident on the device (keeps its tensors alive)."""

    def __init__(self, struct, tensors):
        self.struct = struct
        self._keep = tensors


def device_packet(pkt, device="cuda", *, gates: bool = False, f32_latents: bool = False) -> DevicePacket:
    """Upload a host packet (harness.synth.Packet-like) in trainer-state or COO form."""
    t = {}
    t["lat"] = torch.from_numpy(np.ascontiguousarray(pkt.latents_f32 if f32_latents else pkt.latents)).to(device)
    t["dec"] = torch.from_numpy(np.ascontiguousarray(pkt.decoders, np.float32)).to(device) if pkt.decoders.size else \
        torch.zeros(1, dtype=torch.float32, device=device)
    kw = dict(n=pkt.n, n_pad=pkt.n_pad, sh_degree=pkt.deg, lat_dim=pkt.lat, latents=t["lat"], decoders=t["dec"],
              latent_kind=QUEEN_LAT_F32 if f32_latents else QUEEN_LAT_INT8, gate=pkt.gate)
    if gates:
        t["la"] = torch.from_numpy(np.ascontiguousarray(pkt.log_alpha)).to(device)
        t["lp"] = torch.from_numpy(np.ascontiguousarray(pkt.pos_pregate)).to(device)
        s = packet_struct(**kw, pos_kind=QUEEN_POS_GATES, log_alpha=t["la"], pos_pregate=t["lp"])
    else:
        k = int(pkt.coo_idx.shape[0])
        t["idx"] = torch.from_numpy(np.ascontiguousarray(pkt.coo_idx).view(np.int32)).to(device) if k else None
        t["val"] = torch.from_numpy(np.ascontiguousarray(pkt.coo_val, np.float32)).to(device) if k else None
        s = packet_struct(**kw, pos_kind=QUEEN_POS_COO, k=k, pos_idx=t["idx"], pos_val=t["val"])
    return DevicePacket(s, t)


def wire_packet(buf: torch.Tensor, hdr: dict) -> DevicePacket:
    """QueenPacket view of a device-resident wire buffer (packet.py layout).

    The live COO count is read on the device from the header (k_dev), so a buffer
    filled by an NCCL broadcast needs no host round trip; hdr supplies only the
    stream-static fields (n, n_pad, degree, latent dims, k_cap, offsets)."""
    base = buf.data_ptr()
    s = packet_struct(n=hdr["n"], n_pad=hdr["n_pad"], sh_degree=hdr["deg"], lat_dim=hdr["lat"],
                      latents=base + hdr["lat_off"], decoders=base + hdr["dec_off"], latent_kind=QUEEN_LAT_INT8,
                      pos_kind=QUEEN_POS_COO, k=hdr["k_cap"], k_dev=base + wire.K_WORD * 4,
                      pos_idx=base + hdr["idx_off"], pos_val=base + hdr["val_off"])
    if hdr["k_cap"] == 0:
        s.pos_idx = None
        s.pos_val = None
    return DevicePacket(s, [buf])


class EntropyPacket:
    """A device-resident entropy-coded frame packet (packet.py version 2).

    decode(ctx) enqueues the GPU rANS decode of every category (one warp per 8192-symbol
    chunk, bounded by each stream's byte size from the header) into an int8 latent scratch [sum L][n_pad]; `struct` is the queen_packet that
    points at that scratch, the decoders and the COO section (k read on the device), so
    apply = decode(ctx) + queen_apply_frame(struct)."""

    def __init__(self, buf: torch.Tensor, hdr: dict, latents: torch.Tensor | None = None):
        self.buf, self.hdr = buf, hdr
        SL = sum(hdr["lat"])
        self.latents = latents if latents is not None else torch.zeros((max(SL, 1), hdr["n_pad"]), dtype=torch.int8,
                                                                        device=buf.device)
        base = buf.data_ptr()
        self.struct = packet_struct(n=hdr["n"], n_pad=hdr["n_pad"], sh_degree=hdr["deg"], lat_dim=hdr["lat"],
                                    latents=self.latents, decoders=base + hdr["dec_off"], latent_kind=QUEEN_LAT_INT8,
                                    pos_kind=QUEEN_POS_COO, k=hdr["k_cap"], k_dev=base + wire.K_WORD * 4,
                                    pos_idx=base + hdr["idx_off"], pos_val=base + hdr["val_off"])
        if hdr["k_cap"] == 0:
            self.struct.pos_idx = None
            self.struct.pos_val = None

    def decode(self, ctx: Context, stream=None):
        if getattr(self, "_dec_args", None) is None:  # the buffer is fixed: marshal once
            import ctypes as C
            base = self.buf.data_ptr()
            ptrs = [base + self.hdr["ans_off"][c] if self.hdr["lat"][c] else None for c in range(5)]
            # bound each stream by its fixed-capacity section (not this frame's used bytes): a
            # captured graph replays the decode on later packets refilled into the same buffer
            offs = [self.hdr["ans_off"][c] for c in range(5)] + [int(self.hdr.get("total", self.buf.numel()))]
            caps = [(min(o for o in offs[c + 1:] if o > offs[c]) - offs[c]) if self.hdr["lat"][c] else 0
                    for c in range(5)]
            self._dec_args = ((C.c_void_p * 5)(*[C.c_void_p(int(p)) if p else None for p in ptrs]),
                              (C.c_int64 * 5)(*[int(x) for x in caps]),
                              (C.c_int32 * 5)(*[int(x) for x in self.hdr["lat"]]))
        ptrs, caps, dims = self._dec_args
        queen_entropy_decode_frame(ctx, ptrs, caps, dims, self.hdr["n"], self.latents, stream)


class Player:
    """Resident scene on one GPU; renders a fixed set of equally-sized views per frame.

    Views are rendered in batches (one queen_render_views call each).  Optionally, batches are
    spread over `lanes` independent (libqueen context, CUDA stream) pairs, pipelined with
    queen_wait_binned so one batch's binning can run under another's blend.  Measured on the
    N3DV-shaped frame this does NOT pay (the 100k-CTA blend grid holds every SM, so the other
    lane's kernels wait for free slots: 2 lanes 3.77 ms vs 1 lane 3.55 ms), hence lanes=1."""

    def __init__(self, planes, n: int, deg: int, cams, *, device: int = 0, keys_cap: int | None = None,
                 views_per_batch: int | None = None, bg=(0.0, 0.0, 0.0), with_T: bool = False, lanes: int = 1,
                 n_cap: int | None = None):
        self.dev = torch.device(f"cuda:{device}")
        self.device = device
        if isinstance(planes, np.ndarray):
            planes = torch.from_numpy(np.ascontiguousarray(planes, np.float32))
        self.planes = planes.to(self.dev).contiguous()
        if n_cap is not None and n_cap > self.planes.shape[1]:  # room for densification growth
            cap = (int(n_cap) + 3) // 4 * 4
            grown = torch.zeros((self.planes.shape[0], cap), dtype=torch.float32, device=self.dev)
            grown[:, :self.planes.shape[1]] = self.planes
            self.planes = grown
        self._planes_b = None  # densification ping-pong buffer (allocated on first use)
        self.n, self.deg = n, deg
        self.cams = list(cams)
        W, H = self.cams[0].width, self.cams[0].height
        if any(c.width != W or c.height != H for c in self.cams):
            raise ValueError("all views of a Player must share width/height")
        self.W, self.H = W, H
        V = len(self.cams)
        vmax = min(V, views_per_batch or QUEEN_MAX_VIEWS, QUEEN_MAX_VIEWS)
        nbatch = (V + vmax - 1) // vmax
        if lanes > 1 and nbatch < lanes and V >= lanes:
            nbatch = lanes  # one batch per lane at least, so binning and blending pipeline across lanes
        self.vpb = (V + nbatch - 1) // nbatch  # balanced batches (e.g. 46 views -> 23 + 23)
        self.batches = [(b, min(b + self.vpb, V)) for b in range(0, V, self.vpb)]
        self.cam_arrays = [camera_array(self.cams[a:b]) for a, b in self.batches]
        self.n_lanes = max(1, min(lanes, len(self.batches)))
        self.ctxs = [Context(device) for _ in range(self.n_lanes)]
        self.ctx = self.ctxs[0]
        self.streams = [None] + [torch.cuda.Stream(device=self.dev) for _ in range(self.n_lanes - 1)]
        self.bg = bg
        # step2: the next packet's apply waits for this frame's projection ("projected", its
        # last read of the SoA) or for its whole binning ("binned")
        self.apply_after = "projected"
        self.frame_lanes = 2  # step2: frames in flight, one libqueen context (workspace) each
        self.rgb = torch.empty((V, 3, H, W), dtype=torch.float32, device=self.dev)
        self.T = torch.empty((V, H, W), dtype=torch.float32, device=self.dev) if with_T else None
        self.scene = gaussians_struct(self.planes, n, deg)
        if keys_cap is None:
            keys_cap = min((1 << 30) - 1, max(1 << 16, 8 * n * self.vpb))
        self.keys_cap = int(keys_cap)
        self._carve()

    def _carve(self):
        for c in self.ctxs:
            c.set_workspace(self.planes.shape[1], self.vpb, self.W, self.H, self.keys_cap)

    def apply(self, pkt, stream=None):
        """A_{t-1} -> A_t: (entropy decode, if the packet is coded) + fused decode/apply."""
        if isinstance(pkt, EntropyPacket):
            pkt.decode(self.ctx, stream)
        queen_apply_frame(self.ctx, self.scene, pkt.struct, stream)

    def render(self, stream=None, out=None, rgb8: bool = False):
        """Render every view into `out` (default self.rgb): fp32 [V][3][H][W]; with rgb8=True the
        display format u8 [V][3][H][W] (queen_render_views_rgb8); with a float16 `out` binary16
        (queen_render_views_f16)."""
        rgb = self.rgb if out is None else out
        fn = _out_fn(rgb8, out)
        main = stream if stream is not None else torch.cuda.current_stream(self.dev)
        if self.n_lanes > 1:
            start = torch.cuda.Event()
            start.record(main)
            for s in self.streams[1:]:
                s.wait_event(start)
        prev = None
        for bi, ((a, b), arr) in enumerate(zip(self.batches, self.cam_arrays)):
            k = bi % self.n_lanes
            s = main if k == 0 else self.streams[k]
            if prev is not None and self.n_lanes > 1:
                # pipeline: this batch's binning starts when the previous batch's binning is done,
                # so it runs under the previous batch's blend on the other lane
                queen_wait_binned(prev, s)
            prev = self.ctxs[k]
            fn(self.ctxs[k], self.scene, None, rgb[a:b], None if self.T is None else self.T[a:b], self.bg, s,
               cam_array=arr)
        for s in self.streams[1:]:
            main.wait_stream(s)
        return rgb

    def capture(self, pkt, out=None, rgb8: bool = False, profile: bool = False):
        """Capture one frame step -- (entropy decode +) apply of `pkt` + render of every view --
        into a CUDA graph and return it (torch.cuda.CUDAGraph; .replay() runs the frame with one
        launch).  The packet's buffers, the output and the workspaces are baked in: replay it
        after refilling the same packet buffer (fixed-capacity wire layout, k read on device).
        Call fit_capacity() first (no host sync may happen inside).  profile=True bakes the
        stage profiler's events into the graph: profile_read() after replays returns the stage
        times of each graph's LAST replay."""
        g = torch.cuda.CUDAGraph()
        self.profile(False)
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):  # warm-up outside capture (allocator, lazy init)
            self.apply(pkt)
            self.render(out=out, rgb8=rgb8)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        if profile:
            self.profile(True)
        with torch.cuda.graph(g):
            self.apply(pkt)
            self.render(out=out, rgb8=rgb8)
        self.profile(False)
        return g

    def densify(self, rem_idx, n_rem: int, add_attrs, n_add: int, stream=None):
        """NEXT #2: apply a densification delta after the frame's residuals (queen_densify):
        drop the removed Gaussians (device u32, strictly increasing), append the binary16
        additions (device [P][n_add]); the set is rebuilt in the second buffer, then swapped."""
        n_new = self.n - int(n_rem) + int(n_add)
        if n_new > self.planes.shape[1]:
            raise QueenError(-2, f"densify: {n_new} Gaussians exceed the capacity {self.planes.shape[1]}")
        if self._planes_b is None:
            self._planes_b = torch.empty_like(self.planes)
        dst = gaussians_struct(self._planes_b, n_new, self.deg)
        queen_densify(self.ctx, self.scene, rem_idx, n_rem, add_attrs, n_add, dst, stream)
        self.planes, self._planes_b = self._planes_b, self.planes
        self.n = n_new
        self.scene = dst

    def render_mask(self, subset_idx, k: int | None = None, k_dev=None, out=None, alpha_thresh: float = 1e-3,
                    dilation: int = 48, stream=None):
        """NEXT #3: u8 [V][H][W] masks of the pixels the Gaussian subset
        (device u32 indices, strictly increasing; e.g. a packet's gated COO) reaches with
        accumulated alpha > alpha_thresh, dilated by a dilation x dilation square."""
        k = int(subset_idx.numel()) if k is None else int(k)
        if out is None:
            out = torch.empty((len(self.cams), self.H, self.W), dtype=torch.uint8, device=self.dev)
        for (a, b), arr in zip(self.batches, self.cam_arrays):
            queen_render_mask(self.ctx, self.scene, subset_idx, k, None, out[a:b], alpha_thresh, dilation, k_dev=k_dev,
                              stream=stream, cam_array=arr)
        return out

    def step(self, next_pkt, out=None, rgb8: bool = False, rendered: torch.cuda.Event | None = None,
             ready: torch.cuda.Event | None = None):
        """Pipelined frame step: render the current scene A_t on the current stream and, on a side
        stream, (entropy-)decode next_pkt and apply it (A_t -> A_{t+1}) once this render's
        binning -- the last read of A_t -- is done (queen_wait_binned), i.e. under the blend of
        frame t.  The current stream then waits for the apply, so the next step renders A_{t+1}.
        `rendered` (optional) is recorded on the current stream right after the render; the side
        stream waits for `ready` (optional, e.g. the packet's H2D on a copy stream) before decoding.
        The images are bit-identical to apply(next) after render() (tested)."""
        if self.n_lanes != 1:
            raise ValueError("pipelined steps need a single render lane")
        main = torch.cuda.current_stream(self.dev)
        if not hasattr(self, "_side"):
            # high priority: the decode/apply blocks are dispatched ahead of the blend's queued
            # blocks as SM slots free up, instead of after the whole blend grid
            self._side = torch.cuda.Stream(device=self.dev, priority=-1)
        side = self._side
        side.wait_stream(main)  # the packet (H2D / broadcast) and the previous step are ordered first
        rgb = self.render(out=out, rgb8=rgb8)
        if rendered is not None:
            rendered.record(main)
        if next_pkt is not None:
            with torch.cuda.stream(side):
                if ready is not None:
                    side.wait_event(ready)
                # decode + apply run under the blend only (the binning stages are latency-bound
                # and slow down when shared; measured: decoding from the step's start cost the
                # binning ~60 us per N3DV frame)
                queen_wait_binned(self.ctx, side)
                if isinstance(next_pkt, EntropyPacket):
                    next_pkt.decode(self.ctx, side)
                queen_apply_frame(self.ctx, self.scene, next_pkt.struct, side)
            main.wait_stream(side)
        return rgb

    def step2(self, next_pkt, out=None, rgb8: bool = False, rendered: torch.cuda.Event | None = None,
              ready: torch.cuda.Event | None = None, consumed: torch.cuda.Event | None = None):
        """Two-lane pipelined frame step (eager): like step(), but frame t renders on lane
        t % frame_lanes (2 by default) --
        its own libqueen context (workspace), a high-priority stream for projection + binning and
        a normal-priority stream for the blend (queen_set_blend_stream) -- and the current stream
        does NOT wait for it, so frame t+1's projection and binning (on the other lane) run under
        frame t's blend.  Frame t+1 starts once packet t+1 is applied (after frame t's binning).
        `rendered` is recorded on the blend stream when frame t's image is complete; `out` must
        not be reused before that (out=None: one of two per-lane image buffers, returned; with_T:
        per-lane T buffers, self.T_lanes).  With out=None the returned buffer is rendered into
        again frame_lanes frames later: a caller that reads it on another stream passes
        `consumed`, an event it records after its last read of THIS call's image (before the step
        frame_lanes frames on); that later step's blend waits for it before overwriting the
        buffer.  Call sync_lanes() before reading results on the current stream."""
        if self.n_lanes != 1:
            raise ValueError("two-lane frame steps need a single view-batch lane")
        main = torch.cuda.current_stream(self.dev)
        if not hasattr(self, "_lanes2"):
            # per lane: context, high-priority binning stream, normal-priority blend stream
            lo, hi = torch.cuda.Stream.priority_range()  # (lowest, highest) priority
            self._lanes2 = []
            for k in range(max(2, int(self.frame_lanes))):
                ctx = self.ctx if k == 0 else Context(self.device)
                if k:  # joins self.ctxs: profiled, status-checked and re-carved with the others
                    ctx.set_workspace(self.planes.shape[1], self.vpb, self.W, self.H, self.keys_cap)
                    self.ctxs.append(ctx)
                bs = torch.cuda.Stream(device=self.dev, priority=lo)
                self._lanes2.append((ctx, torch.cuda.Stream(device=self.dev, priority=hi), bs))
            self._lane_t = 0
            self._side = getattr(self, "_side", None) or torch.cuda.Stream(device=self.dev, priority=hi)
            # reused events (a stream wait takes the event's latest record at enqueue time, and
            # each is re-recorded only after its waits are enqueued): cheaper on the host than
            # wait_stream's fresh event per call -- the host cost bounds short multi-GPU frames
            self._ev_main, self._ev_side = torch.cuda.Event(), torch.cuda.Event()
            self._ev_blend = [torch.cuda.Event() for _ in self._lanes2]
            self._last_blend = None  # the previous batch's blend event (ordered completion)
        nl = len(self._lanes2)
        fb = getattr(self, "_frame_t", 0) % nl  # this frame's image buffer (out=None) / consumer fence
        self._frame_t = getattr(self, "_frame_t", 0) + 1
        if out is None or self.T is not None:  # the lanes' blends overlap: per-frame-slot buffers
            if not hasattr(self, "rgb_lanes"):
                self.rgb_lanes = [self.rgb] + [torch.empty_like(self.rgb) for _ in range(nl - 1)]
                self.T_lanes = ([self.T] + [torch.empty_like(self.T) for _ in range(nl - 1)] if self.T is not None
                                else [None] * nl)
        rgb = self.rgb_lanes[fb] if out is None else out
        T = self.T_lanes[fb] if self.T is not None else None
        if not hasattr(self, "_consumed"):
            self._consumed = [None] * nl
        wait_consumed = self._consumed[fb]  # the reader of this slot's previous image is done
        self._consumed[fb] = consumed if out is None else None
        fn = _out_fn(rgb8, out)
        # The lanes rotate per view BATCH (one batch per frame: per frame), so in a multi-batch
        # frame batch b+1's projection + binning run under batch b's blend on another lane.
        # Blends complete in order when there is more than one batch or more than two lanes (each
        # waits for the previous blend; a later, shorter one could otherwise finish first): the
        # last batch's blend then marks the frame complete.  Two lanes with one batch per frame
        # complete in order anyway, and there the blends' tails may overlap.
        ordered = nl > 2 or len(self.batches) > 1
        used = []
        self._ev_main.record(main)  # the frame's apply (and the caller's ordering) first
        for (a, b), arr in zip(self.batches, self.cam_arrays):
            lane = self._lane_t % nl
            self._lane_t += 1
            ctx, ls, bs = self._lanes2[lane]
            ls.wait_event(self._ev_main)
            if wait_consumed is not None:
                bs.wait_event(wait_consumed)
            if ordered and self._last_blend is not None:
                bs.wait_event(self._last_blend)
            queen_set_blend_stream(ctx, bs)  # only for these calls: render() / step() keep one stream
            try:
                fn(ctx, self.scene, None, rgb[a:b], None if T is None else T[a:b], self.bg, ls, cam_array=arr)
            finally:
                queen_set_blend_stream(ctx, None)
            if ordered:
                self._last_blend = self._ev_blend[lane]
                self._last_blend.record(bs)
            if ctx not in [u for u, _ in used]:
                used.append((ctx, bs))
        if rendered is not None:
            rendered.record(bs)  # the last batch's blend (ordered: after every earlier one)
        if next_pkt is not None:
            side = self._side
            side.wait_event(self._ev_main)
            if ready is not None:
                side.wait_event(ready)
            if self.apply_after == "projected":
                # the projection is the render's only read of A_t (binning and blend read the
                # lane's projected records), so the packet decodes at once and A_{t+1} is applied
                # under this frame's binning: the next frame's projection no longer waits for
                # this frame's binning chain (every lane this frame used: the latest projection
                # on each is this frame's)
                if isinstance(next_pkt, EntropyPacket):
                    next_pkt.decode(ctx, side)
                for c, _ in used:
                    queen_wait_projected(c, side)
            else:
                for c, _ in used:
                    queen_wait_binned(c, side)
                if isinstance(next_pkt, EntropyPacket):
                    next_pkt.decode(ctx, side)
            queen_apply_frame(ctx, self.scene, next_pkt.struct, side)
            self._ev_side.record(side)
            main.wait_event(self._ev_side)
        return rgb

    def sync_lanes(self):
        """The current stream waits for both two-lane render streams (step2)."""
        main = torch.cuda.current_stream(self.dev)
        for _, ls, bs in getattr(self, "_lanes2", []):
            main.wait_stream(ls)
            main.wait_stream(bs)

    def capture_step(self, next_pkt, out=None, rgb8: bool = False, profile: bool = False):
        """CUDA graph of one pipelined step (see step()): render of the current scene + decode and
        apply of next_pkt under its blend.  Replaying it advances the scene by one frame."""
        g = torch.cuda.CUDAGraph()
        self.profile(False)
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        saved = self.planes.clone()
        with torch.cuda.stream(side):  # warm-up outside capture (allocator, lazy init)
            self.step(next_pkt, out=out, rgb8=rgb8)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        self.planes.copy_(saved)  # the warm-up advanced the scene: restore it
        if profile:
            self.profile(True)
        with torch.cuda.graph(g):
            self.step(next_pkt, out=out, rgb8=rgb8)
        self.profile(False)
        return g

    def frame(self, pkt: DevicePacket | None, stream=None):
        if pkt is not None:
            self.apply(pkt, stream)
        return self.render(stream)

    def check_status(self, stream=None) -> tuple[int, int]:
        """Synchronise and read every lane's sticky flags: (worst status, largest K requested)."""
        torch.cuda.synchronize(self.dev)
        worst, info = 0, 0
        for c in self.ctxs:
            st, inf = c.check_status(stream)
            if st < 0 and (worst >= 0 or st < worst):
                worst = st
            elif st > 0 and worst == 0:
                worst = st
            info = max(info, inf)
        return worst, info

    def last_error(self) -> str:
        return "; ".join(c.last_error() for c in self.ctxs if c.last_error())

    def profile(self, enable: bool = True):
        for c in self.ctxs:
            c.profile(enable)

    def profile_read(self, reset: bool = True) -> dict:
        tot = {}
        for c in self.ctxs:
            for k, (ms, n) in c.profile_read(reset).items():
                a, b = tot.get(k, (0.0, 0))
                tot[k] = (a + ms, b + n)
        return tot

    def fit_capacity(self, margin: float = 1.3, stream=None):
        """Render once, and grow keys_cap (re-carving the workspaces) until no capacity error."""
        for _ in range(4):
            self.render(stream)
            st, info = self.check_status(stream)
            if st == -5:
                self.keys_cap = min((1 << 30) - 1, int(info * margin) + 1024)
                self._carve()
                continue
            if st < 0:
                raise QueenError(st, self.last_error())
            return self.keys_cap
        raise QueenError(-5, "could not fit key capacity")
