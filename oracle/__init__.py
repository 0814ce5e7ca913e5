"""Oracle package: CPU restatement + reference build. TEST INFRASTRUCTURE ONLY
(importable by tests/, __graft_entry__.smoke() and bench.py's CPU legs)."""
