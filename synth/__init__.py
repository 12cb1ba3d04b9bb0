"""Seeded synthetic input generators (no method arithmetic). See graphs.py."""
from .graphs import CONFIGS, Config, chung_lu, rmat, erdos_renyi, graph_for, features, uniform, weights, bag_of_words  # noqa: F401
