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


def test_measured_model_files_are_reference_consumable():
    """The measured curves stored under profiles/ are per broadcast stage, so
    the reference's own LatencyModel::load_file + find_crossover
    (latency_model.hpp:169-179, tuner.hpp:17-39, run through oracle/_ref)
    reproduce the crossover measured on the box from the fanout totals."""
    import json
    import os

    import oracle_bind as ob
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in (2, 4):
        path = os.path.join(root, "profiles", f"comm_fanout{f}.json")
        doc = json.load(open(path))
        assert doc["fanout"] == f
        measured = doc["sweep"]["crossover_bytes"]
        lo, hi = doc["sweep"]["rows"][0]["bytes"], doc["sweep"]["rows"][-1]["bytes"]
        # our bisection on the model's path totals == the reference's on the same file
        host, dev = tuner.model_path_totals(doc, f)
        ours = tuner.find_crossover(host, dev, lo, hi)
        assert ob.ref_find_crossover_file(path, f, lo, hi) == ours
        # and the model reproduces the measured totals' crossover to within the
        # copy-curve split (the staging copies are separate curves in the model)
        assert ours is not None and abs(math.log2(ours) - math.log2(measured)) < 1.0, (ours, measured)


def test_save_model_round_trips_through_the_reference(tmp_path):
    """tuner.save_model writes per-stage curves: a synthetic box whose fanout-4
    TOTALS cross at a known size yields a file whose reference crossover at
    fanout 4 is that size."""
    import oracle_bind as ob
    sizes = [float(1 << e) for e in range(10, 31)]
    f = 4
    tot_host = [(b, 20e-6 + b / 20e9) for b in sizes]    # cheaper start, less bandwidth
    tot_dev = [(b, 60e-6 + b / 300e9) for b in sizes]
    tiny = [(b, 1e-9 + b * 0) for b in sizes]
    st = tuner.broadcast_stages(f)
    curves = {"host_bcast": [(b, (t - 2e-9) / st) for b, t in tot_host], "device_bcast": [(b, t / st) for b, t in tot_dev],
              "copy_h2d": tiny, "copy_d2h": tiny, "host_path_total": tot_host, "device_path_total": tot_dev}
    p = str(tmp_path / "m.json")
    tuner.save_model(p, curves, fanout=f)
    want = tuner.find_crossover(tot_host, tot_dev, 1024, 1 << 30)
    got = ob.ref_find_crossover_file(p, f, 1024, 1 << 30)
    assert want is not None and abs(got - want) <= max(2, want // 1000)
