"""TEST INFRASTRUCTURE ONLY: the C oracle (drc_oracle.c) and its ctypes
wrapper. Imported by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; never by the product package."""
