"""TEST INFRASTRUCTURE: CPU restatement of the reference prefix-sum path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
