import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O

    O.build()
    return O


def _memoize_large_make(min_vox=1 << 22, keep=2):
    """Several -m gpu tests build the same large host-side synthetic problem
    (e.g. C5 at (64, 1024, 1024): ~40 s of numpy per call).  Keep the last
    ``keep`` such problems and hand them out again; their arrays are made
    read-only so a test that wrote into one would fail instead of leaking
    into the next.  Small problems and device-side synthesis are untouched."""
    import collections

    import numpy as np

    import synth
    import synth.inputs

    raw = synth.inputs.make
    if getattr(raw, "_memoized", False):
        return
    cache = collections.OrderedDict()

    def make(name, shape=None, device=None, **over):
        shp = tuple(shape) if shape is not None else synth.inputs.CONFIGS[name][1]
        if device is not None or over or int(np.prod(shp)) < min_vox:
            return raw(name, shape, device, **over)
        key = (name, shp)
        if key in cache:
            cache.move_to_end(key)
            return cache[key]
        p = raw(name, shape, device)
        for a in (p.medium, p.source):
            if isinstance(a, np.ndarray):
                a.flags.writeable = False
        cache[key] = p
        while len(cache) > keep:
            cache.popitem(last=False)
        return p

    make._memoized = True
    make.__doc__ = raw.__doc__
    synth.inputs.make = make
    synth.make = make


_memoize_large_make()
