"""Pins for the sensor-noise front end (oracle O0; PAPER.md P:275-281, P:350;
SPEC S:202-210; readings c17, c22)."""
import json
import os

import numpy as np
import pytest
from scipy import stats

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    g = json.load(open(os.path.join(GOLD, "philox4x32_10_kat.json")))
    for v in g["vectors"]:
        out = oracle.philox([int(c, 16) for c in v["ctr"]], [int(k, 16) for k in v["key"]])
        assert out == [int(o, 16) for o in v["out"]]


@pytest.mark.parametrize("k,theta", [(3.98, 0.254), (1.0, 2.0), (0.5, 1.5), (12.0, 0.1)])
def test_gamma_sampler_distribution(k, theta):
    """Marsaglia-Tsang (with the k < 1 boost) against the Gamma(k, theta) CDF."""
    g, _ = oracle.noise_samples(40000, seed=123, k=k, theta=theta)
    ks = stats.kstest(g, stats.gamma(k, scale=theta).cdf)
    assert ks.pvalue > 1e-3, ks
    assert abs(g.mean() - k * theta) < 0.02 * k * theta
    assert abs(g.var() - k * theta * theta) < 0.05 * k * theta * theta


def test_additive_normal_distribution():
    _, n = oracle.noise_samples(40000, seed=7)
    ks = stats.kstest(n, stats.norm(-0.231, 0.83).cdf)
    assert ks.pvalue > 1e-3, ks
    # P(n < 0) = Phi(0.231 / 0.83) = 0.61
    assert abs((n < 0).mean() - stats.norm.cdf(0.231 / 0.83)) < 0.01


def test_moment_match_spec():
    """constant input c, 10^6 pixels: mean within 1% of k theta c + mu,
    variance within 3% of c^2 k theta^2 + sigma^2 (before quantisation)."""
    c = 100.0
    clean = np.full((1000, 1000), c)
    _, val = oracle.sensor_noise(clean, seed=2022, f64=True)
    k, th, mu, s = 3.98, 0.254, -0.231, 0.83
    assert abs(val.mean() - (k * th * c + mu)) < 0.01 * (k * th * c + mu)
    assert abs(val.var() - (c * c * k * th * th + s * s)) < 0.03 * (c * c * k * th * th + s * s)


def test_quantisation_and_clamp():
    """c17: round half up, clamp to [0, 255]; scale 0 is the deterministic k*theta*I."""
    clean = np.array([[0.0, 10.0, 100.0, 200.0, 1000.0]])
    u8, val = oracle.sensor_noise(clean, seed=1, f64=True)
    assert np.array_equal(u8, np.clip(np.floor(val + 0.5), 0, 255).astype(np.uint8))
    assert u8[0, 4] == 255
    z, zv = oracle.sensor_noise(clean, seed=1, f64=True, scale=0.0)
    assert np.array_equal(zv, 3.98 * 0.254 * clean)


def test_streams_are_keyed():
    """Deterministic per (seed, frame, view, pixel); different keys differ."""
    clean = np.full((2, 16, 16), 80.0)
    a = oracle.sensor_noise(clean, seed=5)
    assert np.array_equal(a, oracle.sensor_noise(clean, seed=5))
    assert not np.array_equal(a, oracle.sensor_noise(clean, seed=6))
    assert not np.array_equal(a[0], a[1])                            # frames differ
    assert not np.array_equal(a, oracle.sensor_noise(clean, seed=5, view=1))
    # frame0 offsets the frame counter: image 1 of frame0=0 == image 0 of frame0=1
    assert np.array_equal(a[1], oracle.sensor_noise(clean[:1], seed=5, frame0=1)[0])
