"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no neighbour search, no model,
no integrator).  It only draws random numbers and lays out inputs:

* ``synth.nh3``     -- liquid-NH3 boxes (SURVEY.md §8(d) "Synthetic inputs").
* ``synth.weights`` -- random-init weight files (SURVEY.md App. A order); the
                       file is the contract both sides read with their own
                       readers.
* ``synth.configs`` -- the BASELINE.json configs C1..C5 as concrete recipes.
"""
