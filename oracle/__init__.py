"""CPU oracle — TEST INFRASTRUCTURE ONLY (see pot_oracle.hpp header).

Imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, always as the checker."""
