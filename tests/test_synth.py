"""Host-side checks of the seeded input recipe (synth/): no arithmetic of the method here."""
import synth


def test_anomaly_plants_rates_and_determinism():
    assert synth.anomaly_plants(34, 8, 0.0, 1) == {}
    every = synth.anomaly_plants(34, 8, 1.0, 1)
    assert len(every) == 34 * 8 and set(every.values()) == {4.0}
    half = synth.anomaly_plants(34, 8, 0.5, 3)
    assert 0.35 * 272 < len(half) < 0.65 * 272
    # the same decisions on every call (every rank draws them independently)
    assert half == synth.anomaly_plants(34, 8, 0.5, 3)
    # a new round draws afresh
    assert half != synth.anomaly_plants(34, 8, 0.5, 4)
    # nested: a replica planted at rate r is planted at every higher rate (same uniform draw)
    low = synth.anomaly_plants(34, 8, 0.125, 3)
    assert set(low) <= set(half)
