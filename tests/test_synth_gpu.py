"""The seeded input generator (synth/, DESIGN.md s.5): the GPU kernel and the
numpy twin implement the same counter-based recipe.  The uniforms u1, u2 are
exact (24-bit words), so they must agree bit for bit; the derived directions
and roughnesses (sqrt, sin/cos, pow) to a few fp32 ulp."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import synth
    return synth, torch.device("cuda:0")


@pytest.mark.parametrize("recipe,seed", [(0, 1000), (1, 0), (2, 1), (3, 2), (5, 4)])
def test_gpu_generator_matches_numpy_twin(env, recipe, seed):
    synth, dev = env
    n, first = (1 << 16) + 3, (1 << 32) - 7  # across the 32-bit counter carry
    fixed = [0.3, -0.2, 0.93273790530888, 0.05, 0.3] if recipe == 0 else None
    g = synth.fill(recipe, seed, n, first=first, device=dev, fixed=fixed)
    h = synth.fill_numpy(recipe, seed, n, first=first, fixed=fixed)
    for k in ("u1", "u2"):
        np.testing.assert_array_equal(g[k].cpu().numpy(), h[k], err_msg=k)
    for k in ("wi_x", "wi_y", "wi_z", "alpha_x", "alpha_y"):
        a, b = g[k].cpu().numpy().astype(np.float64), h[k].astype(np.float64)
        tol = 4 * np.spacing(np.abs(b).astype(np.float32)).astype(np.float64) + 1e-7
        assert np.all(np.abs(a - b) <= tol), (k, float(np.abs(a - b).max()))
    # unit directions (recipes with sampled wi)
    if recipe != 0:
        w = np.stack([g[k].cpu().numpy() for k in ("wi_x", "wi_y", "wi_z")]).astype(np.float64)
        assert np.abs(np.linalg.norm(w, axis=0) - 1).max() < 1e-6
