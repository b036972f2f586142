"""The host generator (paper_1609_01882_b200/synth.py) is bit-identical to the
oracle's (and therefore, via the GPU parity tests, to the device generator)."""
import numpy as np
import pytest

import oracle
from paper_1609_01882_b200 import synth


@pytest.mark.parametrize("dim,ncent", [(128, 1000), (256, 4096)])
def test_host_generator_matches_oracle(dim, ncent):
    c = synth.gen_centers(160901882, ncent, dim)
    assert np.array_equal(c.view(np.uint32), oracle.gen_centers(160901882, ncent, dim).view(np.uint32))
    for stream, row0 in ((3, 0), (2, 123456789)):
        a = synth.gen_points(160901882, stream, row0, 300, c)
        b = oracle.gen_points(160901882, stream, row0, 300, c)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    a = synth.gen_points(7, 2, 5, 200, c, normalize=True)
    b = oracle.gen_points(7, 2, 5, 200, c, normalize=True)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
