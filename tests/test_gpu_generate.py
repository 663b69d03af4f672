"""On-device input generation: numpy's Philox uniform stream bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,seed", [(1, 1), (7, 2), (1000, 1), (333_333, 12345)])
def test_device_uniform_particles_bitwise(n, seed):
    from paper_2003_01836_b200 import cli
    x, y, z, q = cli.generate_particles_device(n, seed)
    ref = cli.generate_particles(n, seed)
    np.testing.assert_array_equal(x.cpu().numpy(), ref.sources.x)
    np.testing.assert_array_equal(y.cpu().numpy(), ref.sources.y)
    np.testing.assert_array_equal(z.cpu().numpy(), ref.sources.z)
    np.testing.assert_array_equal(q.cpu().numpy(), ref.charges)


def test_device_uniform_empty():
    from paper_2003_01836_b200 import cli
    assert all(t.numel() == 0 for t in cli.generate_particles_device(0, 3))
