"""CPU oracle for the Lightning-2 hot path. TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs, always as the checker or the timed CPU reference -- never by the product
package. See tila_port.py.
"""
