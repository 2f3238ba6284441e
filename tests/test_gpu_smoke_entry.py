"""__graft_entry__.smoke() (the driver's round-end smoke run) passes on the GPU."""

import pytest

pytestmark = pytest.mark.gpu


def test_graft_smoke():
    import __graft_entry__ as g
    g.smoke()
