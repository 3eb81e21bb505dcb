"""CPU tests of the C ABI: the library loads, exports every symbol include/p3.h declares,
and its host planner reproduces the reference plans byte-for-byte (golden CSV hashes)."""

import hashlib
import re
from pathlib import Path

import pytest

from paper_1905_03960_b200 import _lib
from paper_1905_03960_b200.model import LayerSpec, ModelProfile, builtin_profile
from paper_1905_03960_b200.plan import (
    PlanError,
    SliceKey,
    compare_priority,
    make_baseline_plan,
    make_p3_plan,
    plan_from_csv,
    plan_to_csv,
    priority_sort_key,
    validate_plan,
)

HEADER = Path(__file__).resolve().parents[1] / "include" / "p3.h"


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:16]


def declared_functions() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(p3_\w+)\s*\(", text, re.M))


def test_header_symbols_exported():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)


def profile_of(counts, seed=0):
    return ModelProfile("t", seed, tuple(LayerSpec(i, f"L{i}", c, 1, 1) for i, c in enumerate(counts)))


def test_golden_plans(golden):
    counts = {n: builtin_profile(n).param_counts() for n in ("toy3", "resnet50-like", "vgg19-like", "sockeye-like")}
    counts.update(golden["real_counts"])
    for row in golden["plans"]:
        prof = profile_of(counts[row[1]])
        if row[0] == "p3":
            _, name, servers, ms, nslices, h = row
            plan = make_p3_plan(prof, servers, ms)
            assert len(plan.slices) == nslices
            assert sha(plan_to_csv(plan)) == h, row
        else:
            _, name, servers, big, seed, h = row
            assert sha(plan_to_csv(make_baseline_plan(prof, servers, big, seed))) == h, row
    assert plan_to_csv(make_p3_plan(builtin_profile("toy3"), 2)) == golden["plan_csv_toy3_2"]


# known answers of the reference's tests/test_plan.py:35-96
def test_chunking_and_round_robin():
    plan = make_p3_plan(profile_of([120_000]), 1, 50_000)
    assert [s.length for s in plan.slices] == [50_000, 50_000, 20_000]
    assert [s.offset for s in plan.slices] == [0, 50_000, 100_000]
    (s,) = make_p3_plan(profile_of([50_000]), 1, 50_000).slices
    assert (s.offset, s.length) == (0, 50_000)
    assert [s.server for s in make_p3_plan(builtin_profile("toy3"), 2).slices] == [0, 1, 0]
    assert [s.server for s in make_p3_plan(profile_of([25, 20]), 2, 10).slices] == [0, 1, 0, 1, 0]
    assert all(s.priority == s.key.layer_index for s in make_p3_plan(profile_of([10] * 3), 3).slices)


def test_baseline_known_answers():
    assert [s.length for s in make_baseline_plan(profile_of([1_000_000]), 4).slices] == [250_000] * 4
    assert [s.server for s in make_baseline_plan(profile_of([1_000_000]), 4).slices] == [0, 1, 2, 3]
    assert [s.length for s in make_baseline_plan(profile_of([1_000_002]), 4).slices] == [250_000] * 3 + [250_002]
    p = make_baseline_plan(profile_of([1_000_000, 5]), 2)
    assert len(p.slices_of_layer(0)) == 2 and len(p.slices_of_layer(1)) == 1
    a = make_baseline_plan(profile_of([999_999]), 4, rng_seed=77)
    assert a == make_baseline_plan(profile_of([999_999]), 4, rng_seed=77)


def test_errors_and_roundtrip(tmp_path):
    with pytest.raises(PlanError):
        make_p3_plan(profile_of([10]), 0)
    with pytest.raises(PlanError):
        make_p3_plan(profile_of([10]), 1, 0)
    plan = make_p3_plan(builtin_profile("vgg19-like"), 3, 7_000)
    validate_plan(plan, builtin_profile("vgg19-like"))
    assert plan_from_csv(plan_to_csv(plan)) == plan
    assert compare_priority((0, SliceKey(0, 1)), (2, SliceKey(2, 0))) == -1
    assert compare_priority((1, SliceKey(1, 0)), (1, SliceKey(1, 1))) == -1
    assert priority_sort_key(3, SliceKey(3, 4)) == (3, 3, 4)


def test_host_hashing_matches_oracle():
    import numpy as np
    import p3_oracle as O
    from paper_1905_03960_b200.hashing import fnv1a64, splitmix64_mix, splitmix64_stream

    for s, i in [(0, 0), (9, 3), (2**64 - 1, 77)]:
        assert splitmix64_stream(s, i) == O.stream(s, i)
    for x in (0, 1, 12345, 2**64 - 1):
        assert splitmix64_mix(x) == O.mix(x)
    data = np.arange(1000, dtype=np.float32).tobytes()
    assert fnv1a64(data) == O.fnv(data)
    assert fnv1a64(b"") == 0xCBF29CE484222325


def test_compute_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sm = _lib.ctypes.c_int()
    assert _lib.load().p3_device_info(_lib.ctypes.byref(sm), None, None, None) == _lib.P3_ECUDA


def test_graft_entry_importable():
    # the driver imports __graft_entry__ for build() and smoke()
    import importlib.util

    spec = importlib.util.spec_from_file_location("graft_entry", HEADER.parents[1] / "__graft_entry__.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert callable(mod.build) and callable(mod.smoke)
    import py_compile

    py_compile.compile(str(HEADER.parents[1] / "bench.py"), doraise=True)


def test_tools_parse():
    """The measurement tools behind DESIGN.md / profiles/ stay syntactically valid."""
    import ast
    from pathlib import Path

    for f in sorted((Path(__file__).resolve().parents[1] / "tools").glob("*.py")):
        ast.parse(f.read_text(), filename=str(f))
