"""Host-side runner logic (no GPU): pinned CSV formats of runner.hpp and
config validation of run() (runner.hpp:249-268)."""
import pytest

from paper_2007_10196_b200 import configs, runner


def test_emit_table_format():
    rows = [{"grid": 80, "l1": 3.1760e-07, "linf": 5e-07, "wall_seconds": 0.5},
            {"grid": 160, "l1": 9.914e-09, "linf": 1.5e-08, "wall_seconds": 1.25,
             "order_l1": 5.0016, "order_linf": 5.06}]
    assert runner.emit_table(rows) == (
        "grid,l1,l1_order,linf,linf_order,wall_seconds\n"
        "80,3.1760e-07,,5.0000e-07,,5.00000e-01\n"
        "160,9.9140e-09,5.002,1.5000e-08,5.060,1.25000e+00\n")


def test_series_format():
    assert runner.emit_series([{"t": 0.5, "mass": 1.0, "min": -0.25, "max": 2.0}]) == (
        "t,mass,min,max,h2,hlog\n"
        "0.500000,1.0000000000e+00,-2.5000000000e-01,2.0000000000e+00,,\n")


@pytest.mark.parametrize("kw,msg", [
    ({"roots": [5]}, "at least 6 cells"),
    ({"roots": [10, 20], "cfg": "C4"}, "refinement lists"),
])
def test_run_validation(kw, msg):
    cfg = configs.config(kw.pop("cfg", "ex1"))
    with pytest.raises(ValueError, match=msg):
        runner.run(cfg, ctx=object(), **kw)


def test_error_table_examples():
    assert runner.has_error_table(configs.config("ex1"))
    assert runner.has_error_table(configs.config("ex3a"))
    assert not runner.has_error_table(configs.config("C4"))
    assert not runner.has_error_table(configs.config("C2"))  # past the shock at T = 0.5
