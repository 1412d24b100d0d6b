"""First-frame SH "set" decode on the GPU (NEXT #1 completion): frame 0's
high-frequency SH coefficients arrive as an entropy-coded latent matrix + decoder; the GPU
decodes the stream (queen_entropy_decode) and writes D . float(l) into the SH-rest planes
(queen_set_sh_rest).  Bit-exact vs oracle.set_sh_rest (same fmaf chain, R7), other planes and
padding columns untouched; ragged n; dyadic family exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from harness import synth  # noqa: E402


@pytest.mark.parametrize("name,n,dyadic", [("n3dv", 20003, False), ("immersive", 7001, True), ("meetroom", 4096, False)])
def test_first_frame_sh_set_bit_exact(name, n, dyadic):
    import paper_2412_04469_b200 as Q
    cfg = synth.get_config(name)
    sc = synth.make_scene(cfg, n=n)
    ff = synth.make_first_frame_sh(sc, dyadic=dyadic)
    L = ff.latents.shape[0]
    ctx = Q.Context(0)
    ctx.set_workspace(sc.n_pad, 1, 16, 16, 1024)
    stream = Q.queen_entropy_encode(ff.latents, sc.n)
    lat = torch.full((L, sc.n_pad), 99, dtype=torch.int8, device="cuda")
    Q.queen_entropy_decode(ctx, torch.from_numpy(stream).cuda(), L, sc.n, lat)
    planes = torch.from_numpy(sc.planes).cuda()
    dec = torch.from_numpy(ff.decoder).cuda()
    Q.queen_set_sh_rest(ctx, Q.gaussians_struct(planes, sc.n, sc.deg), lat, L, dec)
    assert ctx.check_status()[0] == 0
    got = planes.cpu().numpy()
    ref = oracle.set_sh_rest(sc.planes, sc.n, sc.deg, ff.latents, ff.decoder)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_set_sh_rest_rejects_bad_args():
    import paper_2412_04469_b200 as Q
    ctx = Q.Context(0)
    ctx.set_workspace(8, 1, 16, 16, 1024)
    p0 = torch.zeros((14, 8), dtype=torch.float32, device="cuda")
    lat = torch.zeros((4, 8), dtype=torch.int8, device="cuda")
    dec = torch.zeros((3, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(Q.QueenError):  # degree 0 has no SH-rest
        Q.queen_set_sh_rest(ctx, Q.gaussians_struct(p0, 8, 0), lat, 4, dec)
    p1 = torch.zeros((23, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(Q.QueenError):  # latent dim out of range
        Q.queen_set_sh_rest(ctx, Q.gaussians_struct(p1, 8, 1), lat, 17, dec)
