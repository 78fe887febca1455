"""Test-infrastructure oracle (CPU restatement of the reference hot path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package; the product package never does.  See ancka_cpu.py.
"""
