"""CPU double-precision oracle -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / ``--impl reference`` legs.  Shares no code with the CUDA
product path (``paper_1908_06909_b200``).
"""
