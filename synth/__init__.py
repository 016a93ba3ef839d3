"""Seeded synthetic input generators (no method arithmetic). See synth/gen.py."""
