"""Host-side contract of the certificate selector (certificates.hpp:152-166): argument checks run
before any device work, like the reference's std::invalid_argument throws."""
import pytest

from paper_2605_08123_b200 import band, certificates

SPEC = band.BandSpec(batch=1, heads=1, seq_q=16, seq_k=16, head_dim=32, half_band=4, base_depth=3, tail_depth=2,
                     epsilon=1.0)


def test_selector_rejects_bad_arguments_without_a_gpu():
    with pytest.raises(ValueError):
        certificates.select_tail_depth(None, None, None, None, SPEC, -1.0, 3)
    with pytest.raises(ValueError):
        certificates.select_tail_depth(None, None, None, None, SPEC, 1.0, -1)
    with pytest.raises(ValueError):
        certificates.select_tail_depth(None, None, None, None, SPEC, 1.0, 3, cost=lambda r: -float(r))
    with pytest.raises(band.UnsupportedDepth):
        certificates.select_tail_depth(None, None, None, None, SPEC, 1.0, 9)
