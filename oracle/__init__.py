"""CPU oracle for the neural-shadow-mapping inference hot path.

TEST INFRASTRUCTURE ONLY. Nothing in ``paper_2301_05262_b200`` imports this
package: it is the checker used by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs, never the thing
measured or shipped.

It restates, in numpy, the reference algorithm of the path
(``/root/reference/pkg/src/shadowkit``):

* :mod:`oracle.features` -- ``raster.EmitterView.project`` /
  ``_shadow_lookup`` / ``assemble_features`` and the derived G-buffer planes
  of ``render_gbuffer`` (raster.py:84-94, 222-278).
* :mod:`oracle.network`  -- the forward operators of ``autodiff.py`` and
  ``network.forward`` (autodiff.py:137-329, network.py:98-209).
* :mod:`oracle.producer` -- the ray-cast G-buffer / shadow-map passes that
  produce the path's inputs (raster.py:75-82, 206-242; scene.py:153-163,
  218-441), for small frames.
* :mod:`oracle.blocker`  -- the blocker-search penumbra plane, a build
  extension with no reference implementation (parity unpinned; it reuses
  ``analysis.penumbra_extents``, analysis.py:240-269).

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable
in the build container) on seeded scenes and commits its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this package
against every fixture, plus the reference test-suite's known answers.
"""
