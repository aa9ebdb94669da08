"""Host-side API behaviour that needs no GPU: parameter validation raises the
reference's exception types, FLOP accounting matches pipeline.py:125-141,
shape-drift is rejected like pipeline.py:286-293, and the package refuses to
run without the CUDA library instead of falling back to the CPU."""

import numpy as np
import pytest
import torch

import paper_2604_18348_b200 as P
from paper_2604_18348_b200.errors import ContractError, ParameterError


def test_count_flops_closed_form():
    L, D, C, Gq, it = 100, 8, 10, 5, 7
    fc = P.count_flops(L, D, C, Gq, density=0.5, kmeans_iters=it, mode="sparse")
    assert fc.flops_full == 4 * L * L * D
    assert fc.flops_sparse == 4 * L * 0.5 * L * D
    assert fc.flops_overhead == 2 * L * C * D * it + L * D + 4 * Gq * C * D
    full = P.count_flops(64, 8, 4, 2, density=0.1, kmeans_iters=0, mode="full")
    assert full.flops_sparse == full.flops_full and full.flops_overhead == 0
    with pytest.raises(ParameterError):
        P.count_flops(0, 8, 4, 2, 0.5, 0, "sparse")


def test_params_validation():
    with pytest.raises(ParameterError):
        P.PipelineParams(scorer="bogus").validate()
    with pytest.raises(ParameterError):
        P.PipelineParams(n_max=10, m0=20).validate()
    with pytest.raises(ParameterError):
        P.PipelineParams(full_layer_quota=1.5).validate()


def test_denoise_input_contracts():
    with pytest.raises(ParameterError):
        P.run_denoise_steps([], P.PipelineParams())
    x = np.zeros((8, 4), np.float32)
    bad = [[[(x, x, x)]], [[(x[:-1], x, x)]]]
    with pytest.raises(ContractError):
        P.run_denoise_steps(bad, P.PipelineParams(full_layer_quota=0.0))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="CUDA"):
        P.kmeans(np.random.default_rng(0).normal(size=(20, 4)).astype(np.float32), 3, seed=0)
