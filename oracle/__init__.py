"""CPU oracle package -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg. The product
package (paper_2405_20067_b200) never imports it; see ndg_oracle.py for the reference citations and
the parity-pinning statement.
"""
