"""ORACLE / TEST INFRASTRUCTURE ONLY.  Importable only from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs — never from the product package."""
