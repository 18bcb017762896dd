"""The spsumma-style CLI (paper_2504_06408_b200/cli.py, mirroring
proj/tools/spsumma.cpp + report.hpp).  CPU: flag parsing, the report and
sweep-table layouts, the --check-oracle host product against the oracle,
verify-corpus.  GPU: `multiply --check-oracle` and `sweep` end to end."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_bind as ob
from paper_2504_06408_b200 import cli, errors, generators
from paper_2504_06408_b200.formats import coo_to_csr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse_flags():
    assert cli.parse_gen("rmat:10:16:1") == (10, 16.0, 1)
    for bad in ("rmat:10:16", "er:1:2:3", "rmat:x:16:1"):
        with pytest.raises(errors.MalformedInputError):
            cli.parse_gen(bad)
    assert cli.parse_thresholds("0,65536,inf") == [0, 65536, cli.K_INF]
    assert cli.parse_thresholds("1,,2") == [1, 2]
    with pytest.raises(errors.MalformedInputError, match="non-numeric threshold 'x'"):
        cli.parse_thresholds("1,x")
    with pytest.raises(errors.MalformedInputError, match="lists no thresholds"):
        cli.parse_thresholds(",")
    with pytest.raises(errors.MalformedInputError, match="--comm expects host, device, or hybrid"):
        cli.parse_comm("nvlink")
    with pytest.raises(errors.MalformedInputError, match="exactly one of --matrix or --gen"):
        cli.load_input(0, "", "")


def _led(scale):
    return {"sim": {p: scale * (i + 1) for i, p in enumerate(cli.PHASES)},
            "wall": {p: 2 * scale * (i + 1) for i, p in enumerate(cli.PHASES)},
            "host_bcasts": 3, "device_bcasts": 5, "bytes_host_path": 100, "bytes_device_path": 1 << 20}


def test_report_layout():
    rep = {"matrix": "rmat:8:4:1", "semiring": "tropical_i32", "procs": 4, "comm": "hybrid",
           "threshold": cli.K_INF, "rows": 256, "cols": 256, "nnz": 999, "checksum": 0xABC, "oracle": True,
           "iterations": [_led(1e-3), _led(3e-3)]}
    lines = cli.report_text(rep).splitlines()
    assert lines[:8] == ["spsumma multiply report", "matrix: rmat:8:4:1", "semiring: tropical_i32", "procs: 4",
                         "comm: hybrid threshold_bytes=inf", "iterations: 2 timed (after 1 untimed warm-up)",
                         "result: rows=256 cols=256 nnz=999 checksum=0000000000000abc", "oracle: PASS"]
    assert lines[8] == "first_iteration:"
    assert lines[9] == "  first prepare: sim=0.001000000 wall=0.002000000"
    assert lines[14] == "  first payload_bcasts: host=3 device=5 bytes_host=100 bytes_device=1048576"
    assert lines[15] == "mean_over_timed_iterations:"
    assert lines[16] == "  mean prepare: sim=0.002000000 wall=0.004000000"
    assert len(lines) == 22
    tab = cli.sweep_table_text([{"threshold": 0, "pct_host": 0.0, "comm_s": 1e-4, "local_s": 2e-3, "checksum": 7},
                                {"threshold": cli.K_INF, "pct_host": 100.0, "comm_s": 2e-4, "local_s": 2e-3,
                                 "checksum": 7}]).splitlines()
    assert tab[0] == "threshold_bytes\tpct_host_bcasts\tsim_comm_seconds\twall_local_seconds\tresult_checksum"
    assert tab[1] == "0\t0.00\t0.000100000\t0.002000000\t0000000000000007"
    assert tab[2].startswith("inf\t100.00\t")


@pytest.mark.parametrize("sr", [0, 1, 2, 4])
def test_check_oracle_host_product_matches_oracle(sr):
    m = generators.generate_rmat(sr, 8, 8.0, 3)
    i, j, v = cli.host_product(m)
    a = coo_to_csr(m)
    want = ob.orc_multiply(ob.Mat.of(a), ob.Mat.of(a))
    wi = np.repeat(np.arange(want.nrows), np.diff(want.ptr))
    assert np.array_equal(i, wi) and np.array_equal(j, want.idx)
    assert cli.values_close(sr, v, want.vals)


def test_verify_corpus_subcommand(capsys):
    assert cli.main(["verify-corpus"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].startswith("PASS rmat generator (65536x65536")
    assert out[1:] == ["SKIP atmosmodd (no file supplied)", "SKIP delaunay (no file supplied)",
                       "SKIP long (no file supplied)"]


def test_errors_exit_1(capsys):
    assert cli.main(["multiply", "--gen", "bad"]) == 1
    assert "error: " in capsys.readouterr().err


def _cli(*args):
    env = dict(os.environ, PYTHONPATH=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_2504_06408_b200.cli", *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


@pytest.mark.gpu
def test_multiply_check_oracle_on_gpu():
    r = _cli("multiply", "--gen", "rmat:10:16:1", "--semiring", "tropical_i32", "--iters", "2", "--check-oracle")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert "oracle: PASS" in lines
    m = generators.generate_rmat(4, 10, 16.0, 1)
    a = coo_to_csr(m)
    want = ob.orc_multiply(ob.Mat.of(a), ob.Mat.of(a))
    assert f"result: rows=1024 cols=1024 nnz={want.nnz} checksum={ob.orc_checksum(want):016x}" in lines
    assert any(x.startswith("  mean local_multiply: sim=") for x in lines)


@pytest.mark.gpu
def test_sweep_on_gpu():
    r = _cli("sweep", "--gen", "rmat:9:8:2", "--semiring", "boolean", "--sweep", "0,inf")
    assert r.returncode == 0, r.stderr
    rows = [x.split("\t") for x in r.stdout.splitlines()[1:]]
    assert [x[0] for x in rows] == ["0", "inf"]
    assert rows[0][4] == rows[1][4]  # same C at every threshold
