"""The reference's black-box operator stand-ins on the device (SURVEY §8(f)
row 2): glu_cu_apply_operator against SimOperator::apply / apply_operator
(simop.cpp:16-41, 120-132) of the reference build, bit for bit, and the fused
"edit T-down, then upsample" entry point (glu_cu_apply_operator_field) against
the reference's apply_field(field, apply_operator(op, low)).

Tolerance: none.  (Gamma uses the device pow, at most 2 ulp in double from
the true value, like glibc's: the float results agree unless the double lies
within a few ulp of a float rounding midpoint, ~2^-27 per value; the seeded
inputs below exercise ~10^6 values.)"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _lr_image():
    """A C4-sized LR image (480 x 270) plus edge values: exact 0 / 1, values
    outside [0, 1] (clamped), and exact zeros that make negative-coefficient
    mixes produce -0.0."""
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(480, 270, 4, 0)
    rng = np.random.default_rng(9)
    img[:4] = rng.random((4, 480, 3), dtype=np.float32) * 1.6 - 0.3
    img[4, :, :] = 0.0
    img[5, :, :] = 1.0
    img[6, ::2, :] = 0.0
    return np.ascontiguousarray(img)


def _ops(glu):
    m = np.array([[0.9, 0.1, -0.05], [-0.2, 1.1, 0.05], [0.0, -0.3, 1.2]])
    neg = -np.abs(m)  # all-negative rows: -0.0 from zero pixels
    return [("identity", glu.glu.identity_op(), 0, {}),
            ("gain", glu.glu.scalar_gain_op(0.5), 1, {"gain": 0.5}),
            ("gain_clamp", glu.glu.scalar_gain_op(1.7), 1, {"gain": 1.7}),
            ("mix", glu.glu.channel_mix_op(m.reshape(9)), 2, {"mix": m}),
            ("mix_neg", glu.glu.channel_mix_op(neg.reshape(9)), 2, {"mix": neg}),
            ("gray", glu.glu.grayscale_op(), 3, {}),
            ("gamma_inv", glu.glu.gamma_op(1 / 2.2), 4, {"gamma": 1 / 2.2}),
            ("gamma", glu.glu.gamma_op(2.2), 4, {"gamma": 2.2}),
            ("invert", glu.glu.invert_op(), 5, {})]


def test_apply_operator_matches_reference(glu, reference):
    img = _lr_image()
    dev = torch.from_numpy(img).cuda()
    for name, op, kind, kw in _ops(glu):
        got = glu.glu.apply_operator(op, dev).cpu().numpy()
        want = reference.apply_operator(kind, img, **kw)
        assert got.tobytes() == want.tobytes(), name
    # the configs' operator chains: gamma(1/2.2) then channel_mix (C2 / C4), mix only (C5)
    from paper_2307_09582_b200 import workloads
    for seed in (1002, 1004, 1005):
        M = workloads.gamma_mix_op(seed).M
        g = glu.glu.apply_operator(glu.glu.gamma_op(1 / 2.2), dev)
        got = glu.glu.apply_operator(glu.glu.channel_mix_op(M.reshape(9)), g).cpu().numpy()
        want = reference.apply_operator(2, reference.apply_operator(4, img, gamma=1 / 2.2), mix=M)
        assert got.tobytes() == want.tobytes(), seed


def test_parse_operator_and_validation(glu):
    G = glu.glu
    assert G.parse_operator("gain:0.25").gain == 0.25
    assert G.parse_operator("mix:1,0,0,0,1,0,0,0,1").kind == G.SimOperator.Kind.ChannelMix
    assert G.parse_operator("gray").linear() and not G.parse_operator("gamma:2").linear()
    for bad, msg in (("mix:1,2", "mix needs 9"), ("mix:1,0,0,0,1,0,0,0,1,5", "exactly 9"),
                     ("blur", "unknown operator"), ("gain:-1", "gain must be >= 0"),
                     ("gamma:0", "gamma must be > 0")):
        with pytest.raises(ValueError, match=msg):
            G.parse_operator(bad)


@pytest.mark.parametrize("clamp", [True, False])
def test_fused_operator_apply_matches_reference(glu, reference, clamp):
    """glu_cu_apply_operator_field == apply_field(field, apply_operator(op, low))
    on a joint-optimised field (the C5 edit loop), every operator kind."""
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(1280, 720, 5, 0)
    r = glu.joint_optimize(torch.from_numpy(img).cuda(), 8)
    low = r.low.cpu().numpy()
    P = r.field.numpy()
    for name, op, kind, kw in _ops(glu):
        got = glu.glu.apply_operator_field(r.field, op, r.low, clamp).cpu().numpy()
        want = reference.apply_field(P, 8, reference.apply_operator(kind, low, **kw), clamp)
        assert got.tobytes() == want.tobytes(), (name, clamp)


def test_matte_operator_matches_numpy_stand_in(glu):
    """The C3 matte (harness operator, BASELINE.json configs[2]) on the device
    equals the numpy expression bench.py's CPU baseline uses."""
    from paper_2307_09582_b200 import workloads
    img = _lr_image()
    got = glu.op_matte(torch.from_numpy(img).cuda()).cpu().numpy()
    assert got.tobytes() == workloads.matte_numpy(img).tobytes()
