"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs
(cpu_baseline and --impl reference), as the checker / the CPU baseline.  The
product package (paper_2311_12716_b200) never imports, links or calls it.
"""
