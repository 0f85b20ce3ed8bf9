"""JSON text exactly as the reference writes it: nlohmann::json::dump(2).

The reference's objects are std::map-backed, so keys come out sorted.
Doubles use the shortest round-trip digits, with the same fixed/exponent
switch as nlohmann's dtoa (fixed for decimal exponents in (-4, 15],
"1e-05" / "1e+16" style otherwise). That is Python's repr(float) layout.
Integral doubles keep a ".0". inf/NaN are written as null. Strings are
UTF-8, not \\u-escaped.
"""
from __future__ import annotations

import json
import math


def _clean(o):
    if isinstance(o, float):
        return None if (math.isnan(o) or math.isinf(o)) else o
    if isinstance(o, dict):
        return {k: _clean(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_clean(v) for v in o]
    return o


def dumps(obj) -> str:
    return json.dumps(_clean(obj), indent=2, sort_keys=True, ensure_ascii=False,
                      separators=(",", ": "), allow_nan=False)


def dumps_compact(obj) -> str:
    """nlohmann::json::dump() without indent."""
    return json.dumps(_clean(obj), sort_keys=True, ensure_ascii=False, separators=(",", ":"),
                      allow_nan=False)
