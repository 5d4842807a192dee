"""Seeded synthetic inputs (no method arithmetic). See inputs/gen.py."""
