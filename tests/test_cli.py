"""CLI surface and exit codes (proj/tools/accosim_main.cpp:4-10, 192-205) —
the parts that need no GPU."""
import json

from paper_2406_02613_b200.__main__ import main


def test_memory_command(capsys):
    assert main(["memory", "--method", "acco", "--k", "12", "--n", "64", "--psi", "7.5e9"]) == 0
    j = json.loads(capsys.readouterr().out)
    assert j["bytes"] == 46.40625e9 and j["gb"] == 46 and j["method"] == "acco"


def test_verify_memory_suite(capsys, tmp_path):
    out = tmp_path / "rep.json"
    assert main(["verify", "--suite", "memory", "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["suite"] == "memory" and rep["pass"] and len(rep["checks"]) == 20
    assert set(rep["checks"][0]) >= {"name", "lhs", "rhs", "slack", "pass"}


def test_exit_codes_for_bad_input(tmp_path, capsys):
    assert main([]) == 2
    assert main(["bogus"]) == 2
    assert main(["verify", "--suite", "zero-bubble"]) == 2
    assert main(["memory", "--method", "pipedream"]) == 2
    assert main(["run", "--config", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"problem": {"kind": "gpt"}, "method_name": "zero-bubble",
                               "optimizer": {"kind": "adamw", "learning_rate": 0.1}, "t_updates": 3}))
    assert main(["run", "--config", str(bad)]) == 2
    quad = tmp_path / "quad.json"  # analytic problems stay on the CPU oracle, not the B200 path
    quad.write_text(json.dumps({"problem": {"kind": "quadratic"}, "method_name": "acco",
                                "optimizer": {"kind": "sgd", "learning_rate": 0.1}, "t_updates": 3}))
    assert main(["sweep", "--config", str(quad), "--seeds", "1,2"]) == 2
    assert main(["--help"]) == 0
