"""Run-report / scaling-series harness, modelled on the
reference's tests/test_cli.py: argument validation names the offending flag,
reports validate against the report schema, series CSV layout, exit codes.

CPU tests: validation, parsers, the restated schema pinned against the
reference's shipped report_schema.json (when /root/reference is present, i.e.
in the build container), and a report from stubbed counters validating.
GPU tests: every mode builds through libhxf.so and the report validates; the
counters and K norm match the CPU oracle.
"""

import csv
import io
import json
import os

import jsonschema
import numpy as np
import pytest

from paper_1401_6961_b200 import harness as H
from paper_1401_6961_b200.basis import InvalidArgumentError
from paper_1401_6961_b200.exchange import SymmetryCounters, TraversalCounters

REF_SCHEMA = "/root/reference/pkg/src/hexfock/report_schema.json"


@pytest.mark.parametrize("field,value,flag", [
    ("tau_2e", -1.0, "--tau-2e"), ("tau_ovlp", -1.0, "--tau-ovlp"), ("leaf_size", 0, "--leaf-size"),
    ("mode", "bogus", "--mode"), ("bound", "bogus", "--bound"), ("order", "bogus", "--order"),
    ("threads", 0, "--threads"), ("reference", "bogus", "--reference"),
    ("system", "water:abc", "--system"), ("system", "water:0", "--system"), ("system", "nonsense", "--system"),
    ("system", "xyz:", "--system"), ("density", "exp:gamma=abc", "--density"),
    ("density", "exp:beta=1", "--density"), ("density", "nonsense", "--density"),
    ("density", "file:", "--density"),
])
def test_validation_names_flag(field, value, flag):
    with pytest.raises(InvalidArgumentError) as err:
        H.RunConfig(**{field: value}).validate()
    assert flag in str(err.value)


def test_main_exit_codes(capsys):
    assert H.main(["--tau-2e", "-1"]) == 2
    assert "--tau-2e" in capsys.readouterr().err
    assert H.main(["--system", "water:abc"]) == 2
    assert H.main(["--series", "3,2"]) == 2
    assert H.main(["--series", "1,x"]) == 2
    assert H.main(["--series", ","]) == 2


def test_series_argument_checks():
    for sizes in ([3, 2], [2, 2], []):
        with pytest.raises(InvalidArgumentError):
            H.scaling_series(H.RunConfig(), sizes, io.StringIO())


@pytest.mark.skipif(not os.path.exists(REF_SCHEMA), reason="reference tree not present")
def test_schema_restatement_pinned_to_reference():
    with open(REF_SCHEMA) as fh:
        assert H.load_report_schema() == json.load(fh)


def test_series_columns():
    assert H.SERIES_COLUMNS[:9] == ["n", "n_functions", "mode", "tau_2e", "tau_ovlp", "wall_seconds",
                                    "eri_quartets", "leaf_contractions", "tasks_culled"]
    assert H.SERIES_COLUMNS[-1] == "naive_symmetry_time_ratio"
    assert len(H.SERIES_COLUMNS) == 9 + 9 + 1


def test_xyz_and_density_parsers(tmp_path):
    xyz = tmp_path / "s.xyz"
    xyz.write_text("3\ncomment\nO 0 0 0\nH 0.96 0 0\nH -0.24 0.93 0\n")
    sysm = H.load_xyz(str(xyz))
    assert [a.element for a in sysm.atoms] == ["O", "H", "H"]
    assert np.allclose(sysm.atoms[1].position, [0.96 * 1.8897259886, 0, 0])
    assert sysm.n_functions > 3
    bad = tmp_path / "b.xyz"
    bad.write_text("2\n\nH 0 0 0\n")
    with pytest.raises(H.FormatError):
        H.load_xyz(str(bad))
    bad.write_text("1\n\nH 0 x 0\n")
    with pytest.raises(H.FormatError):
        H.load_xyz(str(bad))
    d = tmp_path / "p.txt"
    d.write_text("2\n1 2\n0 1\n")
    assert np.array_equal(H.load_density_file(str(d)), [[1, 1], [1, 1]])
    d.write_text("2\n1 2 3\n")
    with pytest.raises(InvalidArgumentError):
        H.load_density_file(str(d))


def test_missing_files_are_validation_errors(tmp_path):
    with pytest.raises(InvalidArgumentError):
        H.build_inputs(H.RunConfig(system=f"xyz:{tmp_path}/missing.xyz"))
    with pytest.raises(InvalidArgumentError):
        H.build_inputs(H.RunConfig(system="water:1", density=f"file:{tmp_path}/missing.txt"))


def test_inputs_hilbert_permutes_file_density(tmp_path):
    xyz = tmp_path / "s.xyz"
    xyz.write_text("3\n\nH 4 0 0\nH 0 0 0\nH 2 0 0\n")
    P = np.arange(9.0).reshape(3, 3)
    P = P + P.T
    d = tmp_path / "p.txt"
    d.write_text("3\n" + " ".join(repr(float(v)) for v in P.ravel()) + "\n")
    s_in, _, P_in = H.build_inputs(H.RunConfig(system=f"xyz:{xyz}", density=f"file:{d}", order="input"))
    s_h, _, P_h = H.build_inputs(H.RunConfig(system=f"xyz:{xyz}", density=f"file:{d}", order="hilbert"))
    pos_in = [tuple(sh.center) for sh in s_in.shells]
    perm = [pos_in.index(tuple(sh.center)) for sh in s_h.shells]
    assert np.array_equal(P_h, P_in[np.ix_(perm, perm)])


def test_report_from_stub_counters_validates(monkeypatch):
    def fake(config, mode, system, P):
        if mode == "naive":
            return np.eye(2), TraversalCounters().to_dict(), {c: 0 for c in H.CASE_LABELS}
        if mode == "symmetry":
            d = SymmetryCounters().to_dict()
            return np.eye(2), d, d["case_tasks"]
        return np.eye(2), {}, {c: 0 for c in H.CASE_LABELS}
    monkeypatch.setattr(H, "execute", fake)
    for mode in H.MODES:
        r = H.run(H.RunConfig(system="water:1", mode=mode, reference="dense"))
        jsonschema.validate(r, H.load_report_schema())
        assert r["comparison"]["max_abs_diff"] == 0.0


# ---------------------------------------------------------------- device

@pytest.mark.gpu
@pytest.mark.parametrize("mode", list(H.MODES))
def test_gpu_report_validates(mode):
    r = H.run_report(H.RunConfig(system="water:1", mode=mode, tau_ovlp=0.0))
    jsonschema.validate(r, H.load_report_schema())
    assert r["mode"] == mode and r["k_frobenius"] > 0.0
    if mode in ("dense", "dense-screened"):
        assert all(v == 0 for v in r["case_occurrences"].values())


@pytest.mark.gpu
def test_gpu_report_matches_oracle():
    from oracle import hexfock_oracle as ho
    cfg = H.RunConfig(system="water:3", mode="symmetry", reference="naive")
    r = H.run(cfg)
    jsonschema.validate(r, H.load_report_schema())
    assert r["comparison"]["relative_frobenius"] <= 1e-11
    system, _, P = H.build_inputs(cfg)
    st = ho.Setup(system, P, tau_ovlp=cfg.tau_ovlp, leaf_size=cfg.leaf_size)
    K, c = st.symmetric(cfg.tau_2e)
    for k, v in c.to_dict().items():
        if k == "culled_bound_ledger":
            assert abs(r["counters"][k] - v) <= 1e-12 * max(abs(v), 1e-300)
        else:
            assert r["counters"][k] == v, k
    assert abs(r["k_frobenius"] - np.linalg.norm(K)) <= 1e-12 * np.linalg.norm(K)


@pytest.mark.gpu
def test_gpu_dense_comparison_and_file_inputs(tmp_path):
    r = H.run(H.RunConfig(system="water:1", mode="naive", tau_2e=0.0, tau_ovlp=0.0, reference="dense"))
    assert r["comparison"]["max_abs_diff"] <= 1e-11
    xyz = tmp_path / "s.xyz"
    xyz.write_text("2\n\nH 0 0 0\nH 0.6 0 0\n")
    d = tmp_path / "p.txt"
    d.write_text("2\n1 0\n0 1\n")
    r = H.run(H.RunConfig(system=f"xyz:{xyz}", density=f"file:{d}", mode="naive", tau_2e=0.0,
                          tau_ovlp=0.0, reference="dense"))
    assert r["system"]["n_functions"] == 2 and r["system"]["n_molecules"] is None
    assert r["comparison"]["max_abs_diff"] <= 1e-11


@pytest.mark.gpu
def test_gpu_series_rows(tmp_path):
    out = tmp_path / "s.csv"
    assert H.main(["--series", "1,2", "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert [r["mode"] for r in rows] == ["naive", "symmetry"] * 2
    assert [r["n"] for r in rows] == ["1", "1", "2", "2"]
    for r in rows:
        assert int(r["eri_quartets"]) > 0
        if r["mode"] == "naive":
            assert all(int(r["case_" + c]) == 0 for c in H.CASE_LABELS)
    sym = [r for r in rows if r["mode"] == "symmetry"]
    assert all(sum(int(r["case_" + c]) for c in H.CASE_LABELS) > 0 for r in sym)


def _golden_reports():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reports.json")) as fh:
        return json.load(fh)


def test_golden_reports_validate():
    for case in _golden_reports():
        r = dict(case["report"], generated_at="x", wall_seconds=0.0)
        jsonschema.validate(r, H.load_report_schema())


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(5))
def test_gpu_report_matches_reference_golden(idx):
    """Device report vs the reference harness's own report (tests/golden/make_reports.py)."""
    case = _golden_reports()[idx]
    ref = case["report"]
    r = H.run(H.RunConfig(**case["kwargs"]))
    jsonschema.validate(r, H.load_report_schema())
    assert r["config"] == ref["config"] and r["system"] == ref["system"] and r["mode"] == ref["mode"]
    assert r["case_occurrences"] == ref["case_occurrences"]
    for k, v in r["counters"].items():
        if k == "culled_bound_ledger":
            assert abs(v - ref["counters"][k]) <= 1e-12 * abs(ref["counters"][k])
        else:
            assert v == ref["counters"][k], k
    # the dense-screened twin forms no skipped_bound_sum; every other counter is present
    assert set(ref["counters"]) - set(r["counters"]) <= {"skipped_bound_sum"}
    assert abs(r["k_frobenius"] - ref["k_frobenius"]) <= 1e-12 * ref["k_frobenius"]
    if ref["comparison"] is not None:
        assert r["comparison"]["reference_mode"] == ref["comparison"]["reference_mode"]
        assert r["comparison"]["max_abs_diff"] <= 1e-11
