"""B200-native (sm_100a, fp64) EQP-IFT element core behind the reference's
``ReducedOperator`` API (arXiv 2305.15661; reference package ``strom``)."""

__version__ = "0.1.0"
