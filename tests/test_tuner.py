"""CPU: the measured-threshold tuner follows the reference's tuner contract
(tuner.hpp:17-117, latency_model.hpp:21-185), checked on the reference's own
bundled synthetic model against golden crossovers computed by the reference."""
import math

import numpy as np

from paper_2504_06408_b200 import tuner

GIB = 1024.0 ** 3


def bundled():
    def sample(base, bw):
        return [(float(1 << e), base + (1 << e) / bw) for e in range(32)]
    return {"host_bcast": sample(30e-6, 12 * GIB), "device_bcast": sample(85e-6, 40 * GIB),
            "copy_h2d": sample(8e-6, 20 * GIB), "copy_d2h": sample(8e-6, 20 * GIB)}


def stages(f):
    return (f - 1).bit_length()


def test_crossover_matches_reference_bundled_model(golden):
    m = bundled()
    for fanout, want in zip((2, 3, 4, 8), golden["crossover"]):
        host = lambda b: (tuner.curve_at(m["copy_d2h"], b) + stages(fanout) * tuner.curve_at(m["host_bcast"], b)
                          + tuner.curve_at(m["copy_h2d"], b))
        dev = lambda b: stages(fanout) * tuner.curve_at(m["device_bcast"], b)
        assert tuner.find_crossover(host, dev, 1, 1 << 30) == int(want)


def test_crossover_properties():
    host = [(1.0, 1e-6), (1e9, 1.0)]
    dev = [(1.0, 1e-4), (1e9, 0.1)]
    x = tuner.find_crossover(host, dev, 1, 1 << 30)
    assert x is not None
    assert tuner.curve_at(host, x - 1) < tuner.curve_at(dev, x - 1)
    assert tuner.curve_at(host, x) >= tuner.curve_at(dev, x)
    assert tuner.find_crossover(dev, host, 1, 1 << 30) is None  # no sign change


def test_threshold_ladder_shape():
    lad = tuner.default_threshold_ladder(1 << 18)
    assert lad[0] == 0 and lad[-1] == (1 << 64) - 1
    assert lad == sorted(lad) and (1 << 18) in lad and len(lad) == 12


def test_model_json_round_trip(tmp_path):
    m = bundled()
    curves = dict(m, host_path_total=m["host_bcast"], device_path_total=m["device_bcast"])
    p = tmp_path / "model.json"
    tuner.save_model(str(p), curves)
    import json
    doc = json.load(open(p))
    assert set(doc["curves"]) == {"host_bcast", "device_bcast", "copy_h2d", "copy_d2h"}
    assert doc["curves"]["host_bcast"][3] == [8.0, 30e-6 + 8 / (12 * GIB)]


def test_crossover_warning():
    """crossover_warning (tuner.hpp:43-53): None when the curves cross, the
    reference's text when one path wins everywhere."""
    host = [(1.0, 1e-6), (1e9, 1.0)]
    assert tuner.crossover_warning(host, [(1.0, 1e-5), (1e9, 0.05)]) is None
    msg = tuner.crossover_warning(host, [(1.0, 1e-7), (1e9, 0.05)])
    assert msg and "no host/device crossover" in msg
