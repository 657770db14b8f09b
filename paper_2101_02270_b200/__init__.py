"""paper_2101_02270_b200 -- B200-native batched Newton-Raphson AC power flow.

Host-side mirror of the reference's pipeline (arXiv 2101.02270 / gridbatch):
case parsing and profiles (``case``), Monte-Carlo scenarios (``scenarios``), and
the batched solver (``solver``) that drives libgbnr.so -- C++ symbolic analysis
plus hand-written sm_100a FP64 kernels behind the C ABI in include/gbnr.h.
"""
from .case import GridCase, CaseError, load_case, parse_matpower  # noqa: F401

__all__ = ["GridCase", "CaseError", "load_case", "parse_matpower"]
