"""phylograd-b200: B200-native engine for the linear-time phylogenetic
log-likelihood gradient (arXiv 1905.12146), drop-in for the reference's
LikelihoodEngine hot path.  See DESIGN.md."""
from .api import (ClockGradient, EngineOptions, GradientReport, LikelihoodEngine, RateCategories, RawAlignment,
                  SitePatternAlignment, SubstitutionModel, Tree, branch_lengths_from_clock, clock_likelihood_gradient,
                  compress_codes_gpu, discrete_gamma_categories, node_time_gradient, parse_fasta, parse_newick)
from ._lib import (CudaFailure, InvalidArgument, LogicError, NcclFailure, NewickError, NotSupported, PgError,
                   RuntimeFailure)

__all__ = [
    "ClockGradient", "clock_likelihood_gradient", "NcclFailure",
    "EngineOptions", "GradientReport", "LikelihoodEngine", "RateCategories", "RawAlignment", "SitePatternAlignment",
    "SubstitutionModel", "Tree", "branch_lengths_from_clock", "compress_codes_gpu", "discrete_gamma_categories", "node_time_gradient",
    "parse_fasta", "parse_newick", "CudaFailure", "InvalidArgument", "LogicError", "NewickError", "NotSupported",
    "PgError", "RuntimeFailure",
]
