"""CPU oracle for the multiple-rank-1-lattice sparse FFT hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline -- the product
package ``paper_2006_13053_b200`` never imports, links or executes anything
under ``oracle/``.

Contents
  gather.c     plain-C restatement of the reference's native kernels
  port.py      numpy restatement of the reference's Python-level algorithms
               (DFT, sampling, zero test, gather, Alg. 1/2/4, R1L
               postprocess, host lattice construction, dimension-incremental
               driver), each function citing the reference file:line
  refload.py   loaders for the reference's own compiled Cython core
               (oracle/_ref/, built by ``make -C oracle ref``)

Pinning: tests/test_oracle_golden.py checks this restatement against the
golden vectors in tests/golden/, which tests/golden/make_golden.py produced by
running the reference itself (imported from /root/reference with its compiled
core) in the build container.
"""
