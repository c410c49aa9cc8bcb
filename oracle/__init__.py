"""CPU oracle for the LO-RANSAC PnP hot path — TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithm of the path that
``paper_2601_04185_b200`` runs on the GPU:

* ``oracle.rng``      numpy 2.3.5 ``SeedSequence`` / ``PCG64`` /
                      ``Generator.choice(n, 3, replace=False)`` (the reference
                      calls it at ``pkg/src/visloc/posest.py:243,252``);
* ``oracle.geometry`` pose / quaternion algebra (``geometry.py:79-203``);
* ``oracle.p3p``      resultant-quartic P3P (``p3p.py:57-306``);
* ``oracle.refine``   LM / IRLS refinement (``refine.py:43-230``);
* ``oracle.posest``   MSAC scoring and the LO-RANSAC driver (``posest.py``);
* ``oracle.lift``     confidence gate, depth decode and lift
                      (``localizer.py:87-197``, ``matchio.py:203-218``,
                      ``mapstore.py:122-134``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` and ``--impl reference``) may import this package, and
only as the checker / the timed CPU reference arm.  The product path
(``paper_2601_04185_b200``) never imports it and has no CPU fallback.

Parity pinning: every module is checked against golden vectors produced by
the real reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` in the build container and stores the outputs in
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""
