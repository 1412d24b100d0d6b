"""Host-side logic of the runtime (no GPU): the output-format routing of a render call and the
bench's frame-lane rule."""
import pytest
import torch

from paper_2412_04469_b200 import (queen_render_views, queen_render_views_f16, queen_render_views_rgb8,
                                   queen_render_views_rgb10)
from paper_2412_04469_b200.runtime import _out_fn


def test_output_format_routing():
    V, H, W = 2, 8, 12
    assert _out_fn(False, None) is queen_render_views
    assert _out_fn(False, torch.empty((V, 3, H, W))) is queen_render_views
    assert _out_fn(True, torch.empty((V, 3, H, W), dtype=torch.uint8)) is queen_render_views_rgb8
    assert _out_fn(False, torch.empty((V, 3, H, W), dtype=torch.uint8)) is queen_render_views_rgb8
    assert _out_fn(False, torch.empty((V, 3, H, W), dtype=torch.float16)) is queen_render_views_f16
    assert _out_fn(False, torch.empty((V, H, W), dtype=torch.int32)) is queen_render_views_rgb10
    assert _out_fn("rgb10", torch.empty((V, H, W), dtype=torch.int32)) is queen_render_views_rgb10
    # a display format without a matching out tensor is an error, not a silent fp32 render
    with pytest.raises(ValueError):
        _out_fn(True, None)
    with pytest.raises(ValueError):
        _out_fn("f16", torch.empty((V, 3, H, W)))
    with pytest.raises(ValueError, match=r"\[V\]\[H\]\[W\]"):
        _out_fn("rgb10", None)


def test_rgb10_packing_rule_matches_header():
    """The R10G10B10A2 word documented in include/queen.h (r | g << 10 | b << 20 | 3 << 30, each
    channel round-half-even(clamp(x, 0, 1) * 1023)) decodes back within 1/2 LSB = 4.9e-4."""
    x = torch.linspace(-0.1, 1.1, 2001, dtype=torch.float32)
    q = torch.round(torch.clamp(x, 0, 1) * 1023.0).to(torch.int64)
    word = q | (q << 10) | (q << 20) | (3 << 30)
    assert int(word.max()) < 2 ** 32
    dec = ((word >> 10) & 1023).double() / 1023.0
    assert float((dec - torch.clamp(x, 0, 1).double()).abs().max()) <= 0.5 / 1023 + 1e-12
