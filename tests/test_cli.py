"""NEXT-1: the paper's example program rng_b200 (n i -> 8*n*i raw bytes on stdout)
and NEXT-2's chart tool.  CPU tests check argument handling and failure without a GPU; the
gpu tests check the byte stream against the oracle and the Fig. 3 summary on stderr."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1609_01257_b200 as P
from paper_1609_01257_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    P.lib()
    return _build.build_cli()


def run(cli, *args, **kw):
    return subprocess.run([cli, *map(str, args)], capture_output=True, timeout=kw.get("timeout", 120))


def test_cli_usage(cli):
    r = run(cli, "--help")
    assert r.returncode == 0 and r.stdout == b"" and b"usage: rng_b200 n i" in r.stderr
    for bad in [(0, 10), (16, 0), ((1 << 32) + 1, 1), ("x", 2), (16,), (16, 2, "--mode", "Z9")]:
        r = run(cli, *bad)
        assert r.returncode == 2 and r.stdout == b"", bad


def test_cli_fails_loudly_without_gpu(cli):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = run(cli, 16, 2)
    assert r.returncode == 1 and r.stdout == b"" and b"CUDA" in r.stderr


def test_plot_events_svg(tmp_path):
    t = tmp_path / "ev.tsv"
    t.write_text("Main\t0\t1000\tINIT_KERNEL\nMain\t1000\t5000\tRNG_KERNEL\nComms\t1000\t9000\tREAD_BUFFER\n"
                 "Host\t9000\t9500\tOUT\n")
    svg = tmp_path / "c.svg"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "plot_events.py"), str(t), str(svg), "--title",
                    "x"], check=True)
    s = svg.read_text()
    assert s.startswith("<svg") and s.count("<rect") >= 4 + 3 and "READ_BUFFER" in s and ">Comms<" in s


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["O2", "O1", "O3", "S0", "S1"])
def test_cli_stream_matches_oracle(cli, mode, golden):
    """Config 1 through the program: stdout is exactly the Eq. 1 byte stream."""
    r = run(cli, 1024, 8, "--mode", mode, "--batch", 3)
    assert r.returncode == 0, r.stderr
    assert len(r.stdout) == 8 * 1024 * 8
    assert hashlib.sha256(r.stdout).hexdigest() == golden("survey_appendix_a.json")["config1_n1024_i8"]["0"]["sha256"]


@pytest.mark.gpu
def test_cli_seed_and_profile(cli, tmp_path):
    exp = tmp_path / "ev.tsv"
    r = run(cli, 5000, 6, "--seed", "0x0123456789ABCDEF", "--profile", "--export", exp, "--batch", 2)
    assert r.returncode == 0, r.stderr
    got = np.frombuffer(r.stdout, dtype="<u8").reshape(6, 5000)
    assert np.array_equal(got, oracle.stream(5000, 6, 0x0123456789ABCDEF))
    err = r.stderr.decode()
    assert " Aggregate times by event  :" in err and "READ_BUFFER" in err and "Time spent in device" in err
    rows = exp.read_text().splitlines()
    assert sum(1 for l in rows if l.endswith("\tREAD_BUFFER")) == 3
    assert sum(1 for l in rows if l.endswith("\tRNG_KERNEL")) == 3 and rows[0].endswith("\tINIT_KERNEL")


@pytest.mark.gpu
def test_cli_closed_pipe_is_an_error(cli):
    p = subprocess.Popen([cli, str(1 << 20), "50"], stdout=subprocess.PIPE, stderr=subprocess.PIPE)
    p.stdout.read(4096)
    p.stdout.close()
    assert p.wait(timeout=120) == 1


@pytest.mark.gpu
def test_cli_resume_from_iteration(cli):
    """--start K emits iterations K .. K+i-1: the tail of the uninterrupted stream."""
    r = run(cli, 1000, 5, "--start", 12)
    assert r.returncode == 0, r.stderr
    got = np.frombuffer(r.stdout, dtype="<u8").reshape(5, 1000)
    assert np.array_equal(got, oracle.stream(1000, 17, 0)[12:])
