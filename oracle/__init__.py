"""CPU oracle for the SageAttention2++ quantized-attention path -- TEST INFRASTRUCTURE.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg.  The product package never imports this.
"""
