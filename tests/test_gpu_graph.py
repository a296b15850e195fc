"""The kernels are stream-ordered and allocation-free after first use, so a
sequence of API calls can be captured into a CUDA graph and replayed (the
launch-overhead regime of config 1, 2^20 elements: SURVEY.md section 8(d))."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("width", (64, 32))
def test_cuda_graph_capture_replay(width, cuda):
    import torch

    from paper_1502_05216_b200 import Twofold, _lib, api

    L = _lib.ensure_device(cuda.index)
    dt = torch.float64 if width == 64 else torch.float32
    n = 1 << 20
    x0 = torch.empty(n, dtype=dt, device=cuda)
    x1 = torch.empty_like(x0)
    _lib.check(L.tf_generate(_lib.DIST_CODES["exp64" if width == 64 else "exp32"], 1, 0, n,
                             x0.data_ptr(), x1.data_ptr(), None), "gen")
    lib = api(width)
    ref = lib.texp(Twofold(x0, x1))                    # eager (also initialises the kernel)
    r2 = lib.tlog1p(Twofold(ref.value, ref.error))
    outs = [torch.empty_like(x0) for _ in range(4)]
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            lib.texp(Twofold(x0, x1), out=(outs[0], outs[1]))
            lib.tlog1p(Twofold(outs[0], outs[1]), out=(outs[2], outs[3]))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(outs[0], ref.value) and torch.equal(outs[1], ref.error)
    assert torch.equal(outs[2], r2.value) and torch.equal(outs[3], r2.error)
