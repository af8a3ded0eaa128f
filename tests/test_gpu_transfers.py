"""The drop-in call with ordinary (pageable) numpy buffers at a size that takes the
staged transfer path (csrc/xfer.cu: >= 64 MB, worker threads + pinned pieces): the K a
reference-style caller gets back equals, bit for bit, the K of the same build with
device-resident P and K."""

import numpy as np
import pytest
import torch

import paper_1401_6961_b200 as hx
from paper_1401_6961_b200 import configs, exchange

pytestmark = pytest.mark.gpu


def test_pageable_numpy_round_trip_equals_device_buffers():
    cfg = configs.make("c4")                      # 3584 functions: P and K are 103 MB each
    n = cfg.n_functions
    assert n * n * 8 >= 64 << 20
    part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
    P_np = np.array(cfg.P, copy=True)             # pageable host array
    # reference-style call: numpy in, numpy out
    K_np, c_np = hx.build_exchange_symmetric(pairs, hx.build_matrix_tree(P_np, part), tau_2e=cfg.tau_2e)
    assert isinstance(K_np, np.ndarray) and K_np.shape == (n, n)
    # device-resident call
    dev = torch.device("cuda", 0)
    P_dev = torch.from_numpy(P_np).to(dev)
    K_dev = torch.empty((n, n), dtype=torch.float64, device=dev)
    _, c_dev, _ = exchange.run_exchange(pairs, pairs, hx.build_matrix_tree(P_dev, part), cfg.tau_2e, "schwarz",
                                        True, True, None, K_out=K_dev)
    assert c_np.eri_shell_quartets == c_dev.eri_shell_quartets
    assert np.array_equal(K_np, K_dev.cpu().numpy())
    # a view with a row offset (unaligned start) goes through the same path
    big = np.zeros((n + 1, n))
    big[1:] = P_np
    K2, _ = hx.build_exchange_symmetric(pairs, hx.build_matrix_tree(big[1:], part), tau_2e=cfg.tau_2e)
    assert np.array_equal(K2, K_np)
