"""CPU tests of the C-ABI boundary (include/ckf.h / libckf.so): the library
loads, exports every declared symbol, and its host control logic (traces,
partitions, schedules, config validation) is bit-exact with the reference's
golden vectors.  No GPU compute is called here."""
import ctypes as C

import pytest

import paper_2506_15461_b200 as P
from paper_2506_15461_b200 import _native as N
from paper_2506_15461_b200 import api


def test_library_exports_every_header_symbol():
    L = N.lib()
    declared = N.exported_symbols_from_header()
    assert len(declared) > 40
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing


def test_traces_bit_exact_with_reference(goldens):
    g = goldens["failures"]
    for p, s, want in g["p_iter"]:
        assert api.hourly_to_per_iteration(p, s) == want
    for c in g["traces"]:
        text = api.generate_trace(c["seed"], c["p_hour"], c["iter_s"], c["iters"], c["stages"])
        assert text == c["trace"]
        assert api.parse_trace(c["trace"]) == c["trace"]


def test_trace_parse_errors_are_parse_errors():
    for bad in ("", "checkfree-trace v2 seed=1\n", "checkfree-trace v1 bogus=3\n",
                "checkfree-trace v1 seed=1 stages=2,3\n5;2\n",
                "checkfree-trace v1 seed=1 stages=2,3\n5,4\n",          # outside eligible set
                "checkfree-trace v1 seed=1 stages=2,3\n5,2\n4,3\n",     # unsorted
                "checkfree-trace v1 seed=1 stages=2,3\n5,2\n5,2\n"):    # duplicate
        with pytest.raises(P.ParseError):
            api.parse_trace(bad)


def test_consecutive_conflicts():
    text = "checkfree-trace v1 seed=1 p_hour=0 iter_s=120 stages=1,2,3,4,5\n3,2\n3,3\n3,5\n9,1\n9,4\n12,4\n12,5\n"
    assert api.consecutive_conflicts(text) == [(3, 2), (12, 4)]


def test_partitions_and_schedules_bit_exact(goldens):
    g = goldens["partition_schedule"]
    for c in g["partitions"]:
        assert [list(r) for r in api.even_partition(c["layers"], c["stages"])] == [list(r) for r in c["ranges"]]
    for c in g["schedules"]:
        assert api.build_schedule(c["m"], c["swapped_half"], c["s"]) == c["orders"]
    for c in g["schedule_errors"]:
        with pytest.raises(P.ConfigError):
            api.build_schedule(c["m"], c["swapped_half"], c["s"])


def test_experiment_config_validation_mirrors_reference():
    buf = C.create_string_buffer(1 << 16)
    bad = [
        "strategy=checkfree-plus;stages=3;layers=6",      # swap needs s >= 4 (experiment.cpp:52-55)
        "strategy=checkfree-plus;microbatches=3;batch=12",  # even microbatch count
        "strategy=checkfree;layers=10;stages=4",          # neighbour recovery needs uniform partition
        "batch=10;microbatches=4",                        # indivisible batch
        "p-hour=1.0",
        "strategy=bogus",
        "stages=9;layers=8",
    ]
    for kv in bad:
        rc = N.lib().ckf_run_experiment(kv.encode(), b"", 1, buf, len(buf))
        assert rc == N.CKF_E_CONFIG, (kv, rc, N.lib().ckf_last_error())


def test_missing_library_is_a_loud_import_error(tmp_path, monkeypatch):
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(N, "_lib", None)
    with pytest.raises(ImportError):
        N.lib()
