import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdinr.so")


@pytest.fixture(scope="session")
def O():
    """The fp64 oracle (test infrastructure)."""
    from oracle import oracle as _o

    _o.lib()
    return _o


def golden_geom(beam, sub_x=1, n_s=8, **over):
    """Geometry of tests/golden/*.txt (SURVEY 8(c) golden values)."""
    g = dict(beam=beam, n_rows=1, n_cols=4, sub_x=sub_x, sub_z=1, n_s=n_s, sod=4.0, odd=4.0,
             pixel_dx=1.0, pixel_dz=1.0, offset_cx=2.0, offset_cz=0.5, fov_radius=2.0,
             rot_center_x=0.0, z_lo=-1.0, z_hi=1.0, t_lo=0.0, t_hi=0.0)
    g.update(over)
    return g


def read_golden(name):
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line)
    return rows
