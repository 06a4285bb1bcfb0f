"""B200-native entropic partial optimal transport (ASPOT + feasible/tuned
Sinkhorn) behind the reference's pot:: solver API. See DESIGN.md."""
from . import pot  # noqa: F401
