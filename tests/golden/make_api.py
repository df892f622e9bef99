"""Record the reference package's public API (names, call signatures, dataclass
fields, enum members) as a fixture, so tests/test_api_parity.py can check the
drop-in without the reference present.

    NUMBA_CACHE_DIR=/tmp/numba_ref PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_api.py
"""

from __future__ import annotations

import dataclasses
import enum
import importlib
import inspect
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
MODULES = ("core", "simd", "plan", "engine", "bench", "cli")


def describe(obj):
    if inspect.isclass(obj):
        if issubclass(obj, enum.Enum):
            return {"kind": "enum", "members": {m.name: repr(m.value) for m in obj}}
        d = {"kind": "class"}
        if dataclasses.is_dataclass(obj):
            d["fields"] = [f.name for f in dataclasses.fields(obj)]
        methods = {}
        for name, m in inspect.getmembers(obj, predicate=inspect.isfunction):
            if not name.startswith("_") or name == "__init__":
                try:
                    methods[name] = [p for p in inspect.signature(m).parameters]
                except (TypeError, ValueError):
                    pass
        d["methods"] = methods
        return d
    if callable(obj):
        sig = inspect.signature(obj)
        return {"kind": "function",
                "params": [[p.name, p.kind.name, None if p.default is inspect.Parameter.empty else repr(p.default)]
                           for p in sig.parameters.values()]}
    if isinstance(obj, (int, float, str, tuple)):
        return {"kind": "value", "repr": repr(obj)}
    return None


def main():
    api = {}
    top = importlib.import_module("prefixscan")
    api["__all__"] = list(top.__all__)
    for mod in MODULES:
        m = importlib.import_module(f"prefixscan.{mod}")
        entries = {}
        for name, obj in vars(m).items():
            if name.startswith("_"):
                continue
            if getattr(obj, "__module__", m.__name__) not in (m.__name__,) and not isinstance(obj, (int, float, str, tuple)):
                continue  # re-exported from elsewhere
            d = describe(obj)
            if d is not None:
                entries[name] = d
        api[mod] = entries
    with open(os.path.join(HERE, "api_signatures.json"), "w") as f:
        json.dump(api, f, indent=1, sort_keys=True)
    print(f"{sum(len(v) for k, v in api.items() if k != '__all__')} entries")


if __name__ == "__main__":
    main()
