"""CPU tests of the host-side interop the path's callers use (SURVEY.md 8(f)
ranks 3-4): the `# taskweave csr v1` text format (csr.cpp:61-98,
test_bench.cpp:117-145) and the scenario config/CSV contract
(config.cpp, scenario.cpp:177-247)."""
import io

import numpy as np
import pytest

import paper_2602_21897_b200 as P
from paper_2602_21897_b200 import scenario as S


def test_dump_matches_reference_text_bit_for_bit(orc, golden):
    m = orc.stencil(3, 3, 3)
    assert P.dump_csr((m.row_ptr, m.col_idx, m.values)) == str(golden["csr_text_3x3x3"][0])


def test_text_round_trip_exact(orc, ref):
    m = orc.stencil(3, 3, 3)
    vals = m.values.copy()
    vals[5] = 0.1 + 1.0 / 3.0  # full-precision-hostile value (test_bench.cpp:117-130)
    text = P.dump_csr((m.row_ptr, m.col_idx, vals))
    rp, ci, va = P.parse_csr(text)
    assert np.array_equal(rp, m.row_ptr) and np.array_equal(ci, m.col_idx)
    assert np.array_equal(va, vals)
    # the reference itself reads our text and writes the same bytes back
    assert ref.load(text).dump() == text


@pytest.mark.parametrize("text,msg", [
    ("not a header\n1 1\n0 1\n0\n26\n", "header"),            # test_bench.cpp:140-141
    ("# taskweave csr v1\n2 2\n0 1 2\n0 1\n26\n", "truncated"),  # test_bench.cpp:142-143
    ("# taskweave csr v1\nx y\n", "size line"),
    ("# taskweave csr v1\n2 1\n0 2 1\n0\n1\n", "decreases"),
    ("# taskweave csr v1\n1 1\n0 1\n5\n1\n", "out of range"),
])
def test_text_rejects_malformed(text, msg):
    with pytest.raises(P.ConfigError, match=msg):
        P.parse_csr(text)


def test_config_precedence_file_env_flags(tmp_path):
    f = tmp_path / "s.cfg"
    f.write_text("# comment\nnx = 12\nny=7\n  tiles = 4,8\nvariant=tasks\n")
    c = S.ScenarioConfig()
    S.apply_config_file(c, str(f))
    assert (c.nx, c.ny, c.tiles) == (12, 7, [4, 8])
    S.apply_env(c, {"TASKWEAVE_NY": "9", "TASKWEAVE_ITERATIONS": "20"})
    assert (c.ny, c.iterations) == (9, 20)
    S.apply_key(c, "ny", "11")
    assert c.ny == 11
    c.validate()
    assert c.id_for(4) == "cg-tasks-cuda-single-rt-w4-t4"
    c.scenario_id = "exp"
    assert c.id_for(8) == "exp-t8"


@pytest.mark.parametrize("key,value,msg", [
    ("nx", "abc", "expected an integer"), ("variant", "fancy", "unknown value"),
    ("bogus", "1", "unknown config key"), ("tiles", "", "empty list"),
    ("poll_period", "x", "expected a number"),
])
def test_config_rejects(key, value, msg):
    with pytest.raises(P.ConfigError, match=msg):
        S.apply_key(S.ScenarioConfig(), key, value)


def test_config_file_diagnostic_has_line(tmp_path):
    f = tmp_path / "bad.cfg"
    f.write_text("nx=4\nthis line has no equals\n")
    with pytest.raises(P.ConfigError, match=r"bad.cfg:2: expected key=value"):
        S.apply_config_file(S.ScenarioConfig(), str(f))


def test_validate_rules():
    c = S.ScenarioConfig(variant="monolithic", tiles=[4])
    with pytest.raises(P.ConfigError, match="monolithic variant requires tiles=1"):
        c.validate()
    c = S.ScenarioConfig(backend="device-ta")
    with pytest.raises(P.ConfigError, match="backend=cuda"):
        c.validate()


def test_csv_round_trip_and_header():
    rows = [S.MetricsRow("cg-tasks-cuda-single-rt-w4-t4", 0, i, i < 2, 1e-3 / 3 + i, [0.1, 0.2],
                         [0.0, 0.0], [0.0, 0.0], [0.5, 0.25], 14 * 5, 5) for i in range(4)]
    text = S.HEADER + "\n" + "\n".join(S.to_csv_row(r) for r in rows) + "\n"
    assert S.metrics_csv_header() == ("scenario,repetition,iteration,warmup,iter_time,busy,"
                                      "blocked,suspended,idle,tasks_executed,events_polled")
    back = S.parse_metrics_csv(text)
    assert back == rows
    assert S.to_csv_row(rows[1]).split(",")[4] == "%.17g" % rows[1].iter_time
    with pytest.raises(P.ConfigError, match="unexpected header"):
        S.parse_metrics_csv("a,b\n")
    with pytest.raises(P.ConfigError, match="11 comma-separated"):
        S.parse_metrics_csv(S.HEADER + "\nx,0,0\n")
    with pytest.raises(P.ConfigError, match="missing header"):
        S.parse_metrics_csv("")


def test_cli_config_error_exit_code(capsys):
    from paper_2602_21897_b200 import cli
    assert cli.main(["run", "--variant", "nope"]) == 1
    assert cli.main(["keys"]) == 0
    assert "stream_pool" in capsys.readouterr().out
