"""ctypes binding of the reference episode harness (TEST INFRASTRUCTURE ONLY).

oracle/_ref/libkeep_ref_episode.so is oracle/ref_episode_shim.cpp compiled
over the UNMODIFIED reference headers (generate_episode, MemoryStore,
run_episode, compare_csv: harness.hpp / memory_store.hpp).  Text in, text out
in the reference's own JSON / JSONL / CSV formats.  Only tests/ use it, as the
checker of paper_2602_23592_b200.episode.
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libkeep_ref_episode.so")


def available() -> bool:
    return os.path.exists(LIB)


class EpisodeOracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


class EpisodeOracle:
    def __init__(self):
        self.lib = lib = C.CDLL(LIB)
        for n in ("kre_last_error", "kre_output"):
            getattr(lib, n).restype = C.c_char_p
        lib.kre_generate.argtypes = [C.c_char_p]
        lib.kre_run_episode.argtypes = [C.c_char_p] * 3
        lib.kre_compare_csv.argtypes = [C.c_char_p] * 5
        lib.kre_store_replay.argtypes = [C.c_char_p] * 2

    def _call(self, f, *args) -> str:
        rc = f(*[a.encode() for a in args])
        if rc != 0:
            raise EpisodeOracleError(rc, self.lib.kre_last_error().decode())
        return self.lib.kre_output().decode()

    def generate(self, config_json: str) -> str:
        """generate_episode -> trace_to_jsonl."""
        return self._call(self.lib.kre_generate, config_json)

    def run_episode(self, config_json: str, trace_jsonl: str, strategy: str) -> dict:
        return json.loads(self._call(self.lib.kre_run_episode, config_json, trace_jsonl, strategy))

    def compare_csv(self, config_json: str, trace_jsonl: str, strategies, ks=(), rs=()) -> str:
        return self._call(self.lib.kre_compare_csv, config_json, trace_jsonl, ",".join(strategies),
                          ",".join(str(k) for k in ks), ",".join(repr(float(r)) for r in rs))

    def store_replay(self, config_json: str, trace_jsonl: str) -> list:
        return [json.loads(ln) for ln in self._call(self.lib.kre_store_replay, config_json, trace_jsonl).splitlines()]
