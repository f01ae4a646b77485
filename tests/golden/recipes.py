"""Per-run golden recipes (pure data), shared by make_golden.py (reference
side) and the tests (product + oracle side).

Each recipe names a problem/profile the product's ``problems`` module can
rebuild; ``ref_profile`` tells make_golden.py how the reference builds the
same input (its own registry, or a custom profile for the two inputs the
reference lacks).
"""

RUNS = [
    # C1: reference configs/acoustics_pulse.cfg, serial, 100 steps
    dict(name="c1_acoustics_pulse_256_mc_100", problem="acoustics2d", profile="gaussian_pressure",
         options={"amplitude": 1.0, "width": 0.08}, cells=(256, 256), lower=(0.0, 0.0),
         upper=(1.0, 1.0), dtype="float64", bc="reflective", limiter="mc", speed="bound",
         drive=("max_steps", 100)),
    dict(name="c1_frames_to_0.12", problem="acoustics2d", profile="gaussian_pressure",
         options={"amplitude": 1.0, "width": 0.08}, cells=(256, 256), lower=(0.0, 0.0),
         upper=(1.0, 1.0), dtype="float64", bc="reflective", limiter="mc", speed="bound",
         drive=("until", 0.12, (0.06,))),
    # C2 shape: radial dam break, reflective, MC, adaptive dt with reverts
    dict(name="radial_dam_break_64x64_float64", problem="shallow_water2d", profile="radial_dam_break",
         options={}, cells=(64, 64), lower=(-1.0, -1.0), upper=(1.0, 1.0), dtype="float64",
         bc="reflective", limiter="mc", speed="bound", drive=("max_steps", 30)),
    dict(name="radial_dam_break_128x128_float64", problem="shallow_water2d", profile="radial_dam_break",
         options={}, cells=(128, 128), lower=(-1.0, -1.0), upper=(1.0, 1.0), dtype="float64",
         bc="reflective", limiter="mc", speed="bound", drive=("max_steps", 40)),
    dict(name="radial_dam_break_64x48_float32", problem="shallow_water2d", profile="radial_dam_break",
         options={}, cells=(64, 48), lower=(-1.0, -1.0), upper=(1.0, 1.0), dtype="float32",
         bc="reflective", limiter="mc", speed="bound", drive=("max_steps", 30)),
    # engineered under-estimate -> reverts (pkg/tests/test_acceptance.py:287-318 shape)
    dict(name="dam_break_revert_64x16", problem="shallow_water2d", profile="dam_break",
         options={"h_left": 8.0, "h_right": 0.5}, cells=(64, 16), lower=(0.0, 0.0),
         upper=(1.0, 0.25), dtype="float64", bc="outflow", limiter="mc", speed=("scale", 0.6),
         drive=("until", 0.15, ())),
    *[dict(name=f"hump_periodic_32_{lim}", problem="shallow_water2d", profile="gaussian_hump",
           options={}, cells=(32, 32), lower=(0.0, 0.0), upper=(1.0, 1.0), dtype="float64",
           bc="periodic", limiter=lim, speed="bound", drive=("max_steps", 20))
      for lim in ("mc", "minmod", "superbee", "vanleer", "none")],
    *[dict(name=f"acoustics3d_{bc}_{dt}", problem="acoustics3d", profile="gaussian_pressure",
           options={"width": 0.2}, cells=(12, 10, 8), lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0),
           dtype=dt, bc=bc, limiter="superbee", speed="bound", drive=("max_steps", 8))
      for bc in ("reflective", "outflow", "periodic") for dt in ("float64", "float32")],
    # C3 shape: heterogeneous two-material medium (builder extension solver)
    *[dict(name=f"vc_acoustics3d_{dt}", problem="vc_acoustics3d", profile="two_material_pulse",
           options={}, cells=(10, 10, 12), lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0),
           dtype=dt, bc="reflective", limiter="superbee", speed=("value", 1.0),
           drive=("max_steps", 10))
      for dt in ("float64", "float32")],
    *[dict(name=f"advection_square_{n}", problem="advection1d", profile="square",
           options={"left": 0.1, "right": 0.4}, cells=(n,), lower=(0.0,), upper=(1.0,),
           dtype="float64", bc="periodic", limiter="superbee", speed="bound",
           drive=("until", 0.3, (0.1, 0.2)))
      for n in (50, 7)],
    # SW fp32 periodic hump (fp32 parity of the controller)
    dict(name="hump_periodic_48x40_float32", problem="shallow_water2d", profile="gaussian_hump",
         options={"amplitude": 0.8}, cells=(48, 40), lower=(0.0, 0.0), upper=(1.0, 1.0),
         dtype="float32", bc="periodic", limiter="vanleer", speed="bound", drive=("max_steps", 25)),
]
