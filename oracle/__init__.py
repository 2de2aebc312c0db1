"""CPU float64 oracle for the CityGS-X / voxsplat training hot path.

TEST INFRASTRUCTURE ONLY. This package restates, function by function, the
reference algorithm (``/root/reference/pkg/src/voxsplat``) so the CUDA path can
be checked on the same inputs. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it; the
product package never does and has no CPU fallback.

Parity pinning: ``tests/golden/*.npz`` hold outputs of the reference itself
(generated in the build container by ``oracle/make_golden.py``, which imports
``/root/reference``); ``tests/test_oracle_golden.py`` checks this restatement
against them (culling masks, sort order and tile lists bit-exact; float
outputs to 1e-10; gradients to 1e-9 relative).
"""

from .pipeline import (  # noqa: F401
    Cam, adam_update, bin_tiles, cosine_lr, cull, decode, decoder_init, l1_loss,
    depth_l1_loss, normal_l1_loss, project, raster, raster_tile, OracleState, train_step,
    render_view, leaf_gaussians, flatten_decoded, weight_schedule, SPLAT_KEYS,
)
