"""Oracles — TEST INFRASTRUCTURE ONLY.

* oracle.forward : ctypes wrapper of oracle/_build/libforward_oracle.so, the CPU fp32
  restatement of the SLM forward (parity UNPINNED vs the reference, which has no forward;
  its decoder math is pinned to transformers' Llama / Qwen2 code by
  tests/test_oracle_pin_hf.py; see oracle/forward.c header).
* oracle.ref     : ctypes wrapper of oracle/_ref/libagentsim.so, the UNMODIFIED reference
  scheduler compiled from /root/reference/proj/src by oracle/Makefile (the bit-exact
  oracle for scheduling decisions, KV prefix lengths and the trace format).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package.
"""
