"""TEST ORACLE package -- checker only, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this package.  It wraps two shared objects via ctypes:

* ``liboracle.so``           -- the C restatement (comerge_oracle.c);
* ``_ref/libcomerge_ref.so`` -- the unmodified reference library compiled from
  /root/reference/proj (see oracle/Makefile, ref_shim.cpp).
"""
