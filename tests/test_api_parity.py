"""The drop-in exposes the reference's public API: every name, call signature
(parameter names, kinds, defaults), dataclass field and enum member recorded
from the reference by tests/golden/make_api.py must exist here with the same
shape.  Extra names/parameters on our side are allowed only where listed."""

import dataclasses
import enum
import importlib
import inspect
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
API = json.load(open(os.path.join(HERE, "golden", "api_signatures.json")))
PKG = "paper_2312_14874_b200"

# deliberate, documented extensions of the reference's signatures
EXTRA_PARAMS = {
    ("bench", "CaseConfig"): {"device"},               # host / cuda timing (bench.py docstring)
    ("engine", "ScanRequest"): set(),
}
EXTRA_FIELDS = {
    ("bench", "CaseConfig"): {"device"},
    ("bench", "BenchRecord"): {"device", "bandwidth_gbs"},
    ("engine", "RunStats"): {"kernel_launches", "bytes_moved", "reference_plan_only"},
}
# reference entries that are CPU-thread machinery with no GPU counterpart
NOT_PROVIDED = {("engine", "RunStats", "record"), ("engine", "ScanEngine", "_execute")}


def _entries():
    for mod, entries in API.items():
        if mod == "__all__":
            continue
        for name, desc in entries.items():
            yield mod, name, desc


def test_top_level_all_matches():
    ours = importlib.import_module(PKG)
    assert set(API["__all__"]) <= set(ours.__all__)
    for name in API["__all__"]:
        assert hasattr(ours, name), name


@pytest.mark.parametrize("mod,name,desc", list(_entries()), ids=lambda x: x if isinstance(x, str) else "")
def test_public_entry_matches_reference(mod, name, desc):
    m = importlib.import_module(f"{PKG}.{mod}")
    assert hasattr(m, name), f"{mod}.{name} missing"
    obj = getattr(m, name)
    kind = desc["kind"]
    if kind == "value":
        assert repr(obj) == desc["repr"] or mod in ("bench",) and name in ("ALGORITHMS", "CSV_COLUMNS"), \
            f"{mod}.{name} = {obj!r}, reference {desc['repr']}"
        if name in ("ALGORITHMS", "CSV_COLUMNS"):  # the GPU labels / columns are appended, never reordered
            ref = eval(desc["repr"])  # noqa: S307 - a tuple literal from our own fixture
            assert tuple(obj)[:len(ref)] == ref
        return
    if kind == "enum":
        assert issubclass(obj, enum.Enum)
        assert {mm.name: repr(mm.value) for mm in obj} == desc["members"]
        return
    if kind == "function":
        sig = inspect.signature(obj)
        ours = [[p.name, p.kind.name, None if p.default is inspect.Parameter.empty else repr(p.default)]
                for p in sig.parameters.values()]
        assert ours[:len(desc["params"])] == desc["params"], f"{mod}.{name}{sig}"
        for extra in ours[len(desc["params"]):]:
            assert extra[2] is not None or extra[1] in ("VAR_KEYWORD", "VAR_POSITIONAL"), \
                f"{mod}.{name}: extra parameter {extra[0]} must have a default"
        return
    assert kind == "class" and inspect.isclass(obj)
    if "fields" in desc:
        assert dataclasses.is_dataclass(obj), f"{mod}.{name} should be a dataclass"
        fields = [f.name for f in dataclasses.fields(obj)]
        extra = EXTRA_FIELDS.get((mod, name), set())
        assert [f for f in fields if f not in extra] == desc["fields"], f"{mod}.{name} fields {fields}"
    for meth, params in desc["methods"].items():
        if (mod, name, meth) in NOT_PROVIDED:
            continue
        assert hasattr(obj, meth), f"{mod}.{name}.{meth} missing"
        ours = list(inspect.signature(getattr(obj, meth)).parameters)
        extra = EXTRA_PARAMS.get((mod, name), set())
        assert [p for p in ours if p not in extra][:len(params)] == params, f"{mod}.{name}.{meth}{ours}"


def test_install_as_prefixscan_aliases_every_module():
    import subprocess
    import sys
    code = ("import paper_2312_14874_b200 as b; b.install_as_prefixscan(); "
            "import prefixscan, prefixscan.core as c, prefixscan.simd as s; "
            "from prefixscan.engine import ScanRequest; from prefixscan.bench import run_case; "
            "assert prefixscan is b and c.__name__ == 'paper_2312_14874_b200.core'; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         cwd=os.path.dirname(HERE))
    assert out.stdout.strip() == "ok", out.stderr
