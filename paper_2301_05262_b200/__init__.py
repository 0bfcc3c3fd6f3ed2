"""B200-native neural-shadow-mapping inference (arXiv 2301.05262).

Drop-in, GPU-backed replacements for the inference path of the reference
package ``shadowkit``:

* :mod:`.raster`   -- ``assemble_features`` (stage 1 feature pass)
* :mod:`.network`  -- ``NetworkConfig``, ``init_weights``, ``load_network``,
  ``forward`` (stage 2 U-Net) and the :class:`network.Plan` plan layer
* :mod:`.infer`    -- the fused, batched hot path (``ShadowInference``)
* :mod:`.producer` -- GPU G-buffer / shadow-map producers (inputs)
* :mod:`.shard`    -- frame sharding across the GPUs of one node
* :mod:`.scenes`   -- procedural scenes / cameras / emitter frustum fit

All compute runs in ``libnsm.so`` (``include/nsm.h``); importing a module
that needs it raises if the library has not been built.
"""

__version__ = "0.1.0"
