"""TEST INFRASTRUCTURE -- CPU restatement of the reference's algorithm.

Nothing in the product (paper_1811_09736_b200/) imports this package.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use it,
and only as the checker (or as the timed CPU baseline), never as the thing
measured on the GPU or shipped.

Contents:
  oracle.py   numpy restatement of halftile's exact oracle
              (pkg/src/halftile/oracle.py:38-75), the test generators
              (pkg/tests/conftest.py:7-29) and the tile-engine arithmetic of
              the reduction/scan variants (reduce.py / scan.py / engine.py)
  oracle.c    C restatement of the exact oracle (multi-threaded), used as
              the CPU baseline; built by oracle/Makefile into
              oracle/build/liboracle.so
"""
