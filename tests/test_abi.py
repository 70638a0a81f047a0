"""CPU-side checks of the C ABI library: it loads without a GPU, exports every
symbol include/rnntg.h declares, and fails loudly (E_CUDA) when no device is
present -- there is no CPU fallback."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rnntg.h")


@pytest.fixture(scope="module")
def lib():
    so = os.path.join(ROOT, "paper_2406_03791_b200", "librnntg.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "paper_2406_03791_b200", "csrc",
                                                         "Makefile")], check=True)
    from paper_2406_03791_b200 import _lib
    return _lib.lib()


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(rnntg_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    from paper_2406_03791_b200 import _lib
    assert set(_lib.EXPORTS) <= set(names)


def test_abi_version(lib):
    assert lib.rnntg_abi_version() == 1


def test_no_cpu_fallback_without_device(lib):
    if lib.rnntg_device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_2406_03791_b200 import Model, ModelDims, errors
    dims = ModelDims(5, 4, 4, 4, 4)
    with pytest.raises(errors.CudaError):
        Model.from_seed(dims, 1)


def test_dims_validation_maps_to_value_error(lib):
    from paper_2406_03791_b200 import Model, ModelDims, errors
    with pytest.raises(errors.ValueError):
        Model(ModelDims(5, 4, 4, 4, 4, durations=(2, 3)), [np.zeros(s, np.float32) for s in
                                                            ModelDims(5, 4, 4, 4, 4, durations=(2, 3)).param_shapes()])
    with pytest.raises(errors.ValueError):
        Model(ModelDims(5, 4, 4, 4, 4, cell="tanh", layers=2),
              [np.zeros(s, np.float32) for s in ModelDims(5, 4, 4, 4, 4, cell="tanh", layers=2).param_shapes()])


def test_status_codes_match_reference_taxonomy():
    from paper_2406_03791_b200 import errors
    txt = open(HDR).read()
    codes = dict((m.group(1), int(m.group(2))) for m in re.finditer(r"RNNTG_E_([A-Z]+) = (\d+)", txt))
    assert errors.STATUS[codes["VALUE"]] is errors.ValueError
    assert errors.STATUS[codes["DIMENSION"]] is errors.DimensionError
    assert errors.STATUS[codes["INDEX"]] is errors.IndexError
    assert errors.STATUS[codes["STATE"]] is errors.StateError
    assert errors.STATUS[codes["RUNAWAY"]] is errors.RunawayLoopError


def test_synth_matches_oracle_rng():
    from oracle import oracle as O
    from paper_2406_03791_b200 import synth
    d = O.Dims(1024, 640, 640, 640, 1024, (0, 1, 2, 3, 4), O.CELL_LSTM, 2)
    a = O.init_params(1, d)
    b = synth.init_params(1, synth.param_shapes(1024, 640, 640, 640, 1024, (0, 1, 2, 3, 4), "lstm", 2))
    for x, y in zip(a, b):
        assert np.array_equal(x, y.reshape(x.shape))
    assert np.array_equal(O.fill_uniform(2, -1, 1, (4, 7, 9)), synth.encoder_outputs(2, 4, 7, 9))
