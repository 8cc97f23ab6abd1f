"""CPU checker for the GPU engine — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs
may import this package. The product package (paper_2605_09402_b200)
never does; its GPU path fails loudly when the CUDA library is missing.
"""
