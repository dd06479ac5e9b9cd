"""Test-infrastructure oracle (CPU restatement of the reference path).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this."""
