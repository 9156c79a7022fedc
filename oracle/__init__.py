"""CPU parity checkers for the B200 point-convolution library.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package.  The product (``paper_2511_23227_b200``) never imports it.

Two checkers live here:

* ``Oracle``    -- ``liboracle.so``, the C restatement in ``npc_oracle.c`` of the
  reference hot path (every function cites the reference file:line it follows).
* ``Reference`` -- ``_ref/libnpref.so``, the unmodified reference core
  (``/root/reference/proj/core``) compiled from its own sources by
  ``oracle/Makefile``, driven through the ``ref_capi.cpp`` forwarding shim.
"""
from .oracle import Oracle, Reference, OracleError, reference_available  # noqa: F401
