"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain numpy / Python restatement of the reference path
(pkg/src/meshplan: simulator.py execute_serial/global/hierarchical, plan.py
builders, colouring.py, reorder.py) that the tests use as the checker.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it; the product
package never does, and nothing here is ever the thing measured as the
product.  Parity is pinned: ``tests/test_oracle_golden.py`` checks every
function here against golden vectors produced by the real reference
(``tests/golden/make_golden.py``, run in the build container).
"""
