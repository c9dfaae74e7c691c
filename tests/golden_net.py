"""Rebuild the golden-fixture denoiser (tools/make_golden.py:net_and_cond) with the
drop-in create_net, so the GPU box needs no stored weights."""

import numpy as np


def golden_net(arm=None):
    from paper_2410_16727_b200.ref import diffusion, types
    arm = arm or types.default_arm()
    net = diffusion.create_net(diffusion.arch_for_arm(arm), seed=3)
    rng = np.random.default_rng(5)
    for name in list(net.params):
        p = net.params[name]
        net.params[name] = p + 0.02 * rng.standard_normal(p.shape)
    return net
