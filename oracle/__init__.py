"""CPU oracle of the reference algorithms — test infrastructure only.

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU legs; the
product package (paper_2405_05155_b200) never imports it.
"""
