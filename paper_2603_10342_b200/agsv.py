"""ctypes client of the agsv_* ABI (include/agentsim.h) — the reference's scheduler/session
API.  The same class binds either this repo's libagentserve_b200.so (the product) or, in
tests only, the compiled reference library oracle/_ref/libagentsim.so, which is how parity
is checked: identical calls, identical bytes out.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

STATUS = {0: "ok", 1: "invalid_argument", 2: "validation_error", 3: "protocol_error",
          4: "io_error", 5: "no_data", 6: "infeasible"}


class AgsvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_SIG = {
    "agsv_status_name": (C.c_char_p, [C.c_int]),
    "agsv_last_error": (C.c_char_p, []),
    "agsv_string_free": (None, [C.c_void_p]),
    "agsv_config_from_file": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "agsv_config_from_json": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "agsv_config_set_policy": (C.c_int, [C.c_void_p, C.c_char_p]),
    "agsv_config_set_seed": (C.c_int, [C.c_void_p, C.c_uint64]),
    "agsv_config_set_concurrency": (C.c_int, [C.c_void_p, C.c_int]),
    "agsv_config_resolved_json": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_config_free": (None, [C.c_void_p]),
    "agsv_simulate": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_trace_to_file": (C.c_int, [C.c_void_p, C.c_char_p]),
    "agsv_trace_from_file": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "agsv_trace_replay_check": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_trace_workload_hash": (C.c_uint64, [C.c_void_p]),
    "agsv_trace_policy": (C.c_char_p, [C.c_void_p]),
    "agsv_trace_free": (None, [C.c_void_p]),
    "agsv_metrics_summary_json": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_metrics_sessions_csv": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_verify_trace": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "agsv_report_json": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "agsv_report_violation_count": (C.c_int, [C.c_void_p]),
    "agsv_report_vacuous_count": (C.c_int, [C.c_void_p]),
    "agsv_report_assumptions_met": (C.c_int, [C.c_void_p]),
    "agsv_report_free": (None, [C.c_void_p]),
    "agsv_profile_generate": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "agsv_profile_validate": (C.c_int, [C.c_char_p]),
}
SYMBOLS = list(_SIG)


class Agsv:
    """Binding of one agsv_* library."""

    def __init__(self, path: str | Path | None = None):
        if path is None:
            from ._lib import lib
            self.L = lib()
        else:
            self.L = C.CDLL(str(path))
        for n, (res, args) in _SIG.items():
            f = getattr(self.L, n)
            f.restype = res
            f.argtypes = args

    # ---- helpers
    def _check(self, st):
        if st != 0:
            raise AgsvError(st, self.L.agsv_last_error().decode())

    def _take(self, p: C.c_void_p) -> str:
        if not p.value:
            return ""
        s = C.string_at(p.value).decode()
        self.L.agsv_string_free(p)
        return s

    # ---- config
    def config(self, cfg: dict | str) -> "Config":
        text = cfg if isinstance(cfg, str) else json.dumps(cfg)
        h = C.c_void_p()
        self._check(self.L.agsv_config_from_json(text.encode(), C.byref(h)))
        return Config(self, h)

    def run(self, cfg: dict | str) -> "Trace":
        return self.config(cfg).simulate()

    def load_trace(self, path) -> "Trace":
        h = C.c_void_p()
        self._check(self.L.agsv_trace_from_file(str(path).encode(), C.byref(h)))
        return Trace(self, h)

    def profile_generate(self, shape: dict | None = None) -> tuple[str, str | None]:
        out, warn = C.c_void_p(), C.c_void_p()
        self._check(self.L.agsv_profile_generate(json.dumps(shape).encode() if shape else None,
                                                 C.byref(out), C.byref(warn)))
        w = self._take(warn)
        return self._take(out), (w or None)

    def profile_validate(self, doc: dict | str) -> None:
        text = doc if isinstance(doc, str) else json.dumps(doc)
        self._check(self.L.agsv_profile_validate(text.encode()))


class Config:
    def __init__(self, api: Agsv, h):
        self.api, self.h = api, h

    def resolved(self) -> str:
        out = C.c_void_p()
        self.api._check(self.api.L.agsv_config_resolved_json(self.h, C.byref(out)))
        return self.api._take(out)

    def set_policy(self, p: str):
        self.api._check(self.api.L.agsv_config_set_policy(self.h, p.encode()))

    def set_seed(self, s: int):
        self.api._check(self.api.L.agsv_config_set_seed(self.h, s))

    def set_concurrency(self, n: int):
        self.api._check(self.api.L.agsv_config_set_concurrency(self.h, n))

    def simulate(self) -> "Trace":
        h = C.c_void_p()
        self.api._check(self.api.L.agsv_simulate(self.h, C.byref(h)))
        return Trace(self.api, h)

    def __del__(self):
        try:
            self.api.L.agsv_config_free(self.h)
        except Exception:
            pass


class Trace:
    def __init__(self, api: Agsv, h):
        self.api, self.h = api, h

    def save(self, path) -> None:
        self.api._check(self.api.L.agsv_trace_to_file(self.h, str(path).encode()))

    def jsonl(self, tmpdir) -> str:
        p = Path(tmpdir) / f"trace_{id(self)}.jsonl"
        self.save(p)
        return p.read_text()

    def metrics(self) -> dict:
        out = C.c_void_p()
        self.api._check(self.api.L.agsv_metrics_summary_json(self.h, C.byref(out)))
        return json.loads(self.api._take(out))

    def sessions_csv(self) -> str:
        out = C.c_void_p()
        self.api._check(self.api.L.agsv_metrics_sessions_csv(self.h, C.byref(out)))
        return self.api._take(out)

    def replay(self) -> tuple[int, dict]:
        out = C.c_void_p()
        st = self.api.L.agsv_trace_replay_check(self.h, C.byref(out))
        return st, json.loads(self.api._take(out))

    def verify(self, params: dict | None = None) -> tuple[str, int, int, int]:
        """agsv_verify_trace: (report JSON text, violations, vacuous, assumptions_met)."""
        rep = C.c_void_p()
        self.api._check(self.api.L.agsv_verify_trace(self.h, json.dumps(params or {}).encode(), C.byref(rep)))
        try:
            out = C.c_void_p()
            self.api._check(self.api.L.agsv_report_json(rep, C.byref(out)))
            return (self.api._take(out), self.api.L.agsv_report_violation_count(rep),
                    self.api.L.agsv_report_vacuous_count(rep), self.api.L.agsv_report_assumptions_met(rep))
        finally:
            self.api.L.agsv_report_free(rep)

    @property
    def workload_hash(self) -> int:
        return self.api.L.agsv_trace_workload_hash(self.h)

    @property
    def policy(self) -> str:
        return self.api.L.agsv_trace_policy(self.h).decode()

    def __del__(self):
        try:
            self.api.L.agsv_trace_free(self.h)
        except Exception:
            pass
