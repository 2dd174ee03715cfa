"""Parity checkers for the jagged hot path (TEST INFRASTRUCTURE ONLY).

`oracle.restated` wraps oracle/jagged_oracle.c (the plain-C restatement of the reference's
loop nests); `oracle.reference` wraps oracle/_ref/libjagged_ref.so (the reference itself,
compiled from /root/reference sources). Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this package; the product package never does.
"""
