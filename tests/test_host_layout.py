"""Host-side layout of the drop-in result block (CPU; no device work).

`posest._result_block` lays the outputs of one `ransac_pnp` call out as
views of ONE allocation so that a single device-to-host copy returns them
(`_stage_results`).  The views must not overlap, must be 8-byte aligned for
the 8-byte fields, and must have the shapes and dtypes the C ABI writes
(include/visloc_b200.h, vl_ransac_out).
"""

import pytest


@pytest.mark.parametrize("Q,N", [(1, 3), (1, 2000), (7, 12_345), (1000, 50_000_000 // 1000)])
def test_result_block_views(Q, N):
    import torch
    from paper_2601_04185_b200.posest import _result_block
    out = _result_block(Q, N, torch.device("cpu"))
    expect = {"q": ((Q, 4), torch.float64), "t": ((Q, 3), torch.float64), "score": ((Q,), torch.float64),
              "count": ((Q,), torch.int64), "iterations": ((Q,), torch.int64), "stats": ((Q, 4), torch.int64),
              "converged": ((Q,), torch.int32), "flags": ((N,), torch.uint8)}
    assert set(out) == set(expect)
    base = out["q"].untyped_storage().data_ptr()
    spans = []
    for k, (shape, dt) in expect.items():
        v = out[k]
        assert tuple(v.shape) == shape and v.dtype == dt and v.is_contiguous(), k
        assert v.untyped_storage().data_ptr() == base, k  # one allocation
        off = v.data_ptr() - base
        assert off % v.element_size() == 0 and (v.element_size() < 8 or off % 8 == 0), k
        spans.append((off, off + v.numel() * v.element_size(), k))
    spans.sort()
    for (a0, a1, ka), (b0, b1, kb) in zip(spans, spans[1:]):
        assert a1 <= b0, (ka, kb)  # no overlap
    assert spans[-1][1] <= out["q"].untyped_storage().nbytes()
    # writing through one view leaves the others untouched
    for v in out.values():
        v.zero_()
    out["stats"].fill_(-1)
    assert int(out["iterations"].abs().sum()) == 0 and int(out["converged"].abs().sum()) == 0
