"""CPU ORACLE — test infrastructure, NOT product code.

Plain, slow, obviously-correct numpy implementation of what the Computron
(arXiv 2306.13835) hot path computes, written from PAPER.md and the readings in
DESIGN.md.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything from here.  It shares
no code with the CUDA path (`paper_2306_13835_b200/`) and imports nothing from it.

Modules (each function cites the passage it follows):
  weights   C0  counter-based synthetic weights (input spec; not in the paper)
  layout    C2  TP partition + 256-B aligned per-rank arena layout
  checksum  C4  order-independent 64-bit hash (verification; not in the paper)
  swap      C3  chunk-level swap semantics, budget, writeback
  scheduler C1  engine semantics: queues, oldest-head batching, LRU, acks
  forward   C5  OPT forward, exact fp64 and bf16-emulating fp32, TP-simulated (HF OPT)
  metrics   C7  swap latency window, nearest-rank percentiles
  costmodel     alpha-beta transfer closed forms

Pins (tests/test_oracle_*.py) are listed per function in DESIGN.md §Oracle.
"""
