"""relaykv-b200: B200-native RelayCaching relay-prefill engine (arXiv 2603.13289).

The C ABI library librelaykv_b200.so (csrc/) with its Python host mirror
(engine.py, abi.py, hostcache.py, sessions.py) and the C++ drop-in of the
reference's relaykv API (cpp/)."""
