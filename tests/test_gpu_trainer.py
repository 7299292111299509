"""Trainer<float>::fit / evaluate_accuracy parity (training.hpp:50-107): the
device Trainer (host-gather loop and the device-resident epoch loop) against
the REFERENCE's own Trainer<double>::fit (oracle/_ref ref_fit) on the same
dataset -- the seeded shuffle carried across epochs, the smaller last batch,
the mean epoch loss, the final weights -- and the non-finite stop."""
import numpy as np
import pytest

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network, Trainer
from paper_1501_07338_b200.errors import TrainingError
from paper_1501_07338_b200.spec import Precision

from .util import TOL, TOL_STEPS, assert_close

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")]
A = S.Activation

CASES = {
    # 40 samples in batches of 16: two full batches + one of 8, 2 epochs
    "cifar3": (S.cifar3(), 40, 16),
    # MSE targets (values), 10 samples in batches of 4 (4, 4, 2)
    "denoise-mini": (S.NetworkSpec((24, 24, 1), [S.ConvSpec(8, 9, 9, 1, A.relu),
                                                  S.ConvSpec(8, 1, 1, 1, A.relu),
                                                  S.ConvSpec(1, 5, 5, 1, A.identity)],
                                    S.LossKind.mse, 7), 10, 4),
}


def _data(spec, n, seed=5):
    rng = np.random.default_rng(seed)
    h, w, c = spec.input
    imgs = rng.uniform(0, 1, (n, c, h, w)).astype(np.float32)
    if spec.loss == S.LossKind.softmax_ce:
        return imgs, rng.integers(0, spec.output_units(), n).astype(np.int32)
    return imgs, rng.uniform(0, 1, (n, spec.output_units())).astype(np.float32)


@pytest.mark.parametrize("resident", [False, True], ids=["host-loop", "resident"])
@pytest.mark.parametrize("prec", [Precision.tf32x3, Precision.tf32], ids=lambda p: p.name)
@pytest.mark.parametrize("name", list(CASES))
def test_fit_vs_reference_trainer(name, prec, resident):
    spec, n, batch = CASES[name]
    imgs, tg = _data(spec, n)
    is_ce = spec.loss == S.LossKind.softmax_ce
    cfg = S.TrainConfig(lr=0.01, momentum=0.9, batch=batch, epochs=2, seed=3)
    net = Network(spec, batch, prec)
    p0 = net.get_params().astype(np.float64)
    ref_args = (imgs.astype(np.float64), tg if is_ce else None, None if is_ce else tg)
    pr, el, acc = O.ref_fit(spec, p0, *ref_args, cfg.lr, cfg.momentum, batch, cfg.epochs,
                            cfg.seed)
    tr = Trainer(cfg, precision=prec)
    hist = tr.fit(net, imgs, tg, resident=resident)
    tol = TOL[prec]
    assert len(hist) == cfg.epochs
    for e, (a, b) in enumerate(zip(hist, el)):
        assert abs(a - b) <= tol * max(1.0, abs(b)), (e, a, b)
    # final weights: the reference's own float build drifts from its f64 build
    # over the same trajectory; no fp32 path can be held tighter than that
    p32, _, _ = O.ref_fit(spec, p0, *ref_args, cfg.lr, cfg.momentum, batch, cfg.epochs,
                          cfg.seed, f32=True)
    drift = float(np.abs(p32 - pr).max() / np.abs(pr).max())
    assert_close(net.get_params(), pr, max(TOL_STEPS[prec], 2 * drift), "weights after fit")
    if is_ce:
        got = tr.evaluate_accuracy(net, imgs, tg)
        assert abs(got - acc) <= (0.0 if prec == Precision.tf32x3 else 1.0 / n), (got, acc)
    net.close()


def test_nonfinite_stop_resident_equals_host_loop():
    """A non-finite batch loss stops training BEFORE that batch's sgd_step
    (training.hpp:77-80) in both loops: the device-resident loop's guard
    skips the offending update and every later one, so the weights equal the
    host loop's, which raised right after that batch's run_batch."""
    spec, n, batch = S.cifar3(), 40, 16
    imgs, tg = _data(spec, n)
    cfg = S.TrainConfig(lr=0.01, momentum=0.9, batch=batch, epochs=2, seed=3)
    order = list(range(n))
    S.Rng(cfg.seed).shuffle(order)
    # one huge sample in the second batch of epoch 0: its inf activations are
    # zeroed by a ReLU (NaN -> 0, layers.hpp:29), so that batch's loss stays
    # finite but its gradient is not; the NEXT batch's loss is the first
    # non-finite one -- exactly as in the reference, which only checks losses
    imgs[order[20]] = np.float32(3e38)
    res = []
    for resident in (False, True):
        net = Network(spec, batch)
        with pytest.raises(TrainingError, match="non-finite loss at epoch 0, batch 2") as e:
            Trainer(cfg).fit(net, imgs, tg, resident=resident)
        res.append((net.get_params(), str(e.value)))
        net.close()
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][0], res[1][0])
