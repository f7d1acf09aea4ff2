"""CPU parity checker for the RDKV hot path — TEST INFRASTRUCTURE ONLY.

`oracle.load()` returns the C restatement (oracle/liboracle.so);
`oracle.load_ref()` returns the compiled, unmodified reference
(oracle/_ref/librdkv_ref.so). Both expose the same methods (see pylib.py).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
leg import this package; the product path never does.
"""
from .pylib import Config, OracleLib, RefModel, TriZone, build, load, load_ref, ref_available, default_config  # noqa: F401
