"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no GRU, no score, no key,
no cache logic).  It only draws numbers: model parameters (the paper ships
no trained weights) and LibriSpeech-shaped query streams (the
paper's streams come from a live WFST decoder, which is out of
scope).  Both the oracle tests and the GPU path consume exactly these
arrays; see DESIGN.md "Input recipe".
"""
from .model import CONFIGS, ModelDims, generate_model, model_dims
from .workload import Workload, generate_workload

__all__ = ["CONFIGS", "ModelDims", "generate_model", "model_dims",
           "Workload", "generate_workload"]
