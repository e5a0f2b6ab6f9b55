"""The command-line drop-in (paper_2407_02913_b200/sfconv_cli, the reference's
proj/tools/sfconv_cli.cpp over the device path) and the SFCT tensor files.

CPU: option parsing / exit codes (sfconv_cli.cpp:1-5, 198-202, 415-427), catalog export,
validate, configuration errors raised before any device work, SFCT bytes shared between
the C++ and Python writers.  GPU: quantsim and bench against the reference library's own
results for the same seeds (tests/golden/cli_golden.json, made by make_golden.py --cli
through oracle/_ref/cli_golden)."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2407_02913_b200 import sfconv as sc
from paper_2407_02913_b200.sfct import load_sfct, save_sfct

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CLI = os.path.join(ROOT, "paper_2407_02913_b200", "sfconv_cli")
TEST_DROPIN = os.path.join(HERE, "cpp", "test_dropin")
with open(os.path.join(HERE, "golden", "cli_golden.json")) as _f:
    GOLD = json.load(_f)


@pytest.fixture(scope="module", autouse=True)
def built():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2407_02913_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)


def run(args, env=None, timeout=300, cwd=ROOT):
    e = dict(os.environ)
    e.pop("SFC_SEED", None)
    e.update(env or {})
    return subprocess.run([CLI] + list(args), capture_output=True, text=True, timeout=timeout, env=e, cwd=cwd)


# ------------------------------------------------------------------ front end (CPU)
@pytest.mark.parametrize("args", [
    [],                                           # a subcommand is required
    ["frobnicate"],                               # unknown subcommand
    ["quantsim", "--bits", "1"],                  # Range(2, 16)
    ["quantsim", "--bits", "17"],
    ["quantsim", "--channels", "0"],              # PositiveNumber
    ["quantsim", "--padding", "-1"],              # NonNegativeNumber
    ["quantsim", "--size", "abc"],                # conversion error
    ["quantsim", "--bogus", "1"],                 # unexpected option
    ["quantsim", "--bits"],                       # missing value
    ["quantsim", "bench"],                        # one subcommand only
    ["--seed", "-3", "validate"],                 # seed is unsigned
    ["bench", "--reps", "0"],
    ["bench", "--reduced=1"],                     # a flag takes no value
    ["bops"],                                     # --layers is required
    ["quantsim", "--act-scope", "channel"],       # unknown grouping (sfconv_cli.cpp:259-261)
    ["quantsim", "--filter-scope", "tensor"],
    ["quantsim", "--search", "grid"],
    ["quantsim", "--gen", "pink", "--size", "4"],  # unknown generator
    ["quantsim", "--algo", "wino-9x9-3x3"],       # configuration error: unknown algorithm
    ["table1"],                                   # analysis tooling: outside this build
    ["bops", "--layers", "tests/golden/cli_layers.json"],
    ["quantsim", "--layers", "tests/golden/does_not_exist.json"],
    ["quantsim", "--algo", "sfc6-6x6-5x5", "--layers", "tests/golden/cli_layers.json"],  # kernel mismatch
])
def test_usage_and_configuration_errors_exit_2(args):
    r = run(args)
    assert r.returncode == 2, (args, r.stdout, r.stderr)
    assert r.stderr.strip()


def test_help_exits_0():
    r = run(["--help"])
    assert r.returncode == 0
    for sub in ("validate", "table1", "catalog", "quantsim", "bops", "bench", "--seed", "--act-scope", "--reduced"):
        assert sub in r.stdout
    assert run(["quantsim", "--help"]).returncode == 0


def test_error_messages_follow_the_reference():
    r = run(["quantsim", "--algo", "wino-9x9-3x3"])
    assert r.stderr.startswith("configuration error: unknown algorithm")
    r = run(["quantsim", "--algo", "sfc6-6x6-5x5", "--layers", "tests/golden/cli_layers.json"])
    assert r.stderr.strip() == "error: layer 'conv1' kernel 3 does not match algorithm sfc6-6x6-5x5"
    r = run(["quantsim", "--layers", "tests/golden/does_not_exist.json"])
    assert r.stderr.strip() == "error: cannot open layer config: tests/golden/does_not_exist.json"


def test_catalog_export(tmp_path):
    r = run(["catalog"])
    assert r.returncode == 0
    lib_json, lib_hash = sc.catalog_export_json()
    doc = json.loads(r.stdout)
    assert [a["name"] for a in doc["algorithms"]] == ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3",
                                                      "sfc6-6x6-5x5", "sfc6-4x4-7x7"]
    assert r.stdout.strip() == lib_json
    out = tmp_path / "cat.json"
    assert run(["catalog", "--out", str(out)]).returncode == 0
    assert out.read_text() == r.stdout
    # every SFC entry is the reference's own export text (catalog.cpp:562-591)
    with open(os.path.join(HERE, "golden", "catalog_3x3.json")) as f:
        exact = json.load(f)["exact_text"]
    for name, text in exact.items():
        assert text in r.stdout


def test_validate_all_pass():
    r = run(["validate"])
    assert r.returncode == 0, r.stderr
    names = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5", "sfc6-4x4-7x7"]
    assert r.stdout.splitlines() == [f"PASS {n} (8 trials)" for n in names]
    r = run(["--seed", "0x10", "validate", "--algo", "sfc6-7x7-3x3", "--trials", "3"])
    assert r.stdout.splitlines() == ["PASS sfc6-7x7-3x3 (3 trials)"]


def test_malformed_sfc_seed_warns():
    r = run(["validate", "--algo", "sfc4-4x4-3x3", "--trials", "1"], env={"SFC_SEED": "12abc"})
    assert r.returncode == 0
    assert "warning: ignoring malformed SFC_SEED value" in r.stderr


# ------------------------------------------------------------------ SFCT files (CPU)
def test_sfct_python_and_cpp_write_identical_bytes(tmp_path):
    rng = np.random.default_rng(7)
    t = rng.normal(size=(2, 3, 5, 4))
    t.flat[0] = -0.0
    t.flat[1] = 1e-308
    t.flat[2] = np.inf
    a, b = tmp_path / "a.sfct", tmp_path / "b.sfct"
    save_sfct(a, t)
    r = subprocess.run([TEST_DROPIN, "sfct-copy", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert a.read_bytes() == b.read_bytes()
    back = load_sfct(b)
    assert back.shape == t.shape and back.tobytes() == t.tobytes()
    raw = a.read_bytes()
    header = b'{"dtype":"f64","layout":"row-major-nchw","shape":[2,3,5,4]}'
    assert raw[:8] == b"SFCT0001" and raw[8:12] == len(header).to_bytes(4, "little")
    assert raw[12:12 + len(header)] == header and len(raw) == 12 + len(header) + 8 * t.size


@pytest.mark.parametrize("damage,message", [
    (lambda raw: b"NOTSFCT!" + raw[8:], "not an SFCT file"),
    (lambda raw: raw[:10], "truncated SFCT header"),
    (lambda raw: raw[:-10], "truncated SFCT payload"),
    (lambda raw: raw.replace(b'"f64"', b'"f32"'), "unsupported SFCT dtype: f32"),
])
def test_sfct_errors_match_between_python_and_cpp(tmp_path, damage, message):
    a, b = tmp_path / "a.sfct", tmp_path / "b.sfct"
    save_sfct(a, np.arange(24.0).reshape(1, 2, 3, 4))
    a.write_bytes(damage(a.read_bytes()))
    with pytest.raises(RuntimeError, match=message):
        load_sfct(a)
    r = subprocess.run([TEST_DROPIN, "sfct-copy", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 1 and message in r.stdout


# ------------------------------------------------------------------ quantsim / bench (GPU)
def _close(got, want, rel):
    if math.isinf(want) or math.isinf(got):
        return got == want
    return abs(got - want) <= rel * max(abs(want), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["quantsim"], ids=[c["name"] for c in GOLD["quantsim"]])
def test_quantsim_matches_reference(cuda, tmp_path, case):
    """Same seed -> same inputs (mt19937_64 + normal_distribution, onef smoothing) -> the
    reference's report: saturations / values_quantized exact, mse and snr to the fp64
    epilogue's rounding (the real-valued device path keeps vq / uq / pacc bit-exact)."""
    out = tmp_path / "q"
    r = run(case["argv"] + ["--out", str(out)], env=case["env"])
    assert r.returncode == 0, r.stdout + r.stderr
    doc = json.loads((out / "quantsim.json").read_text())
    rows = doc["results"]
    assert [row["layer"] for row in rows] == [g["layer"] for g in case["results"]]
    for row, g in zip(rows, case["results"]):
        assert row["saturations"] == g["saturations"]
        assert row["values_quantized"] == g["values_quantized"]
        assert _close(row["mse"], g["mse"], 1e-9), (row["mse"], g["mse"])
        assert _close(row["snr_db"], g["snr_db"], 1e-9), (row["snr_db"], g["snr_db"])
    # the report text of sfconv_cli.cpp:318-319 (ostream defaults: %g) and the JSON layout
    lines = r.stdout.splitlines()
    for line, row in zip(lines, rows):
        assert line == f"{row['layer']}: snr {row['snr_db']:g} dB, mse {row['mse']:g}, saturated {row['saturations']}"
    assert lines[-1] == f"wrote {out}/quantsim.json"
    m = doc["manifest"]
    assert list(m) == ["catalog_hash", "command", "config_path", "output_dir", "seed"]
    assert m["command"] == "quantsim" and m["seed"] == case["seed"] and m["output_dir"] == str(out)
    assert m["config_path"] == (case["argv"][case["argv"].index("--layers") + 1] if "--layers" in case["argv"] else "")
    assert list(rows[0]) == sorted(rows[0])
    assert (out / "quantsim.json").read_text().startswith('{\n  "manifest": {\n    "catalog_hash": ')


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["bench"], ids=[c["name"] for c in GOLD["bench"]])
def test_bench_gate_and_counters(cuda, case):
    """bench (sfconv_cli.cpp:364-414): fast vs direct agreement gate, then the timing report;
    the product / tile counters per pass equal the reference's (full or paired schedule)."""
    r = run(case["argv"] + ["--reps", "2"])
    assert r.returncode == 0, r.stdout + r.stderr
    fields = {line[:17].strip(): line[17:] for line in r.stdout.splitlines()}
    assert set(fields) == {"algorithm", "agreement", "direct", "tiled", "speedup", "products"}
    assert float(fields["agreement"].split()[0]) <= 1e-10
    assert fields["products"] == f"{case['multiplications']} per pass over {case['tiles']} tiles"
    assert ("paired products" in fields["tiled"]) == ("--reduced" in case["argv"])
    assert float(fields["direct"].split()[0]) > 0 and float(fields["tiled"].split()[0]) > 0
