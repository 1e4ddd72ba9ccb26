"""Test-side alias of the fp32 DiT restatement (oracle/dit_fp32.py)."""
from oracle.dit_fp32 import DiTReference, apply_rope, attention, rms, rope_tables, sinusoid  # noqa: F401
