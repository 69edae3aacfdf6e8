"""NEXT-1: the sampler-only microbenchmark kernels (the paper's GPU methodology,
P:814-817) compute what the float64 oracle replays: per-lane checksums of 64
Listing-1 calls (vndf.h vndf_microbench).  No fix-up runs here, so rare
ill-conditioned samples may exceed the per-sample tolerance; the checksum of a
lane is 64 samples x (1 + 2 + 3) weights, so the bound is 64 * 6 * 2e-5."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", [0, 1, 2], ids=["cap", "heitz", "cap_literal"])
def test_microbench_checksums_match_oracle(method):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import oracle
    import paper_2306_05044_b200 as vndf
    lanes, iters = 1 << 14, 64
    out = torch.empty(lanes, dtype=torch.float32, device="cuda:0")
    vndf.vndf_microbench(method, 11, lanes, iters, out)
    torch.cuda.synchronize()
    ref = oracle.batch_microbench(method, 11, lanes, iters)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    bound = iters * 6 * 2e-5
    assert np.median(err) < 1e-4
    assert (err <= bound).mean() >= (0.999 if method == 0 else 0.99), (err <= bound).mean()
