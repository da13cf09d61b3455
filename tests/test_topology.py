"""CPU tests of the topology / ledger / latency bookkeeping the collectives'
results carry (zs/topology.py), following the reference's test_topology.py
behaviours."""

import pytest


def _zpp():
    import paper_2306_10209_b200 as zpp

    return zpp


def test_links_ranks_and_spans():
    zpp = _zpp()
    from paper_2306_10209_b200.topology import classify_link, span_class

    t = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    assert t.world == 4 and [t.node_of(r) for r in range(4)] == [0, 0, 1, 1]
    assert [classify_link(a, b, t) for a, b in ((0, 1), (0, 0), (0, 2), (3, 1), (2, 3))] == \
        [zpp.INTRA, zpp.INTRA, zpp.INTER, zpp.INTER, zpp.INTRA]
    assert [span_class(s, t) for s in ([0, 1], [2, 3], [1, 2], range(4), [3])] == \
        [zpp.INTRA, zpp.INTRA, zpp.INTER, zpp.INTER, zpp.INTRA]
    assert span_class(range(4), zpp.ClusterTopology(nodes=1, gpus_per_node=4)) == zpp.INTRA
    for bad in (4, -1):
        with pytest.raises(zpp.ValidationError):
            t.node_of(bad)
    for shape in ((0, 2), (2, 0)):
        with pytest.raises(zpp.ValidationError):
            zpp.ClusterTopology(*shape)


def test_ledger_physical_and_volume_rows():
    zpp = _zpp()
    t = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    led = zpp.TrafficLedger()
    led.record_message("ag", 0, 0, t, payload=100)  # a self copy costs nothing
    assert led.physical_bytes() == 0 and led.per_rank == {}
    led.record_message("ag", 0, 1, t, payload=10, metadata=2)
    led.record_message("ag", 0, 2, t, payload=20)
    led.record_message("rs", 1, 3, t, payload=40)
    assert (led.physical_bytes(), led.physical_bytes(label="ag"), led.physical_bytes(cls=zpp.INTER),
            led.physical_bytes(label="ag", cls=zpp.INTRA)) == (70, 30, 60, 10)
    assert led.physical[("ag", zpp.INTRA)].metadata == 2 and led.physical[("ag", zpp.INTRA)].messages == 1
    assert led.labels() == ["ag", "rs"] and led.conservation_holds()

    vol = zpp.TrafficLedger()
    vol.record_volume("ag", zpp.INTER, payload=4000, metadata=40)
    vol.record_volume("rs", zpp.INTER, payload=1000)
    vol.record_volume("rs", zpp.INTRA, payload=700)
    assert (vol.volume_bytes(zpp.INTER), vol.volume_bytes(zpp.INTER, label="ag"),
            vol.volume_bytes(zpp.INTER, label="ag", kind="metadata")) == (5000, 4000, 40)
    assert zpp.normalized_cross_node_volume(vol, 1000) == 2.5
    assert zpp.normalized_cross_node_volume(vol, 1000, label="rs") == 0.5
    with pytest.raises(zpp.ValidationError):
        zpp.normalized_cross_node_volume(vol, 0)

    frozen = zpp.TrafficLedger()
    frozen.record_volume("allgather", zpp.INTER, payload=4000, metadata=40, padding=8)
    frozen.record_volume("reduce_scatter", zpp.INTRA, payload=700)
    assert frozen.to_csv(m_params=1000) == (
        "collective,link_class,payload_bytes,metadata_bytes,padding_bytes,normalized_volume\n"
        "allgather,inter,4000,40,8,2.0\n"
        "reduce_scatter,intra,700,0,0,0.35\n")


def _trace(zpp, im=4, ib=3 * 10**9, em=2, eb=10**9, compute=0.0):
    return zpp.CollectiveTrace(label="x", phases=[zpp.PhaseStats("p", intra_messages=im, intra_bytes=ib,
                                                                 inter_messages=em, inter_bytes=eb,
                                                                 compute_seconds=compute)])


def test_latency_model():
    zpp = _zpp()
    links = zpp.LinkParams(intra_alpha=1e-3, intra_beta=1e9, inter_alpha=1e-2, inter_beta=1e9)
    tr = _trace(zpp)
    one = zpp.estimate_latency(tr, links)
    assert one.intra_seconds == 4e-3 + 3.0 and one.inter_seconds == 2e-2 + 1.0
    assert one.total_seconds == one.intra_seconds + one.inter_seconds
    assert zpp.estimate_latency(tr, links, overlap=False, stages=4).total_seconds == one.total_seconds
    free = zpp.LinkParams(intra_alpha=0.0, intra_beta=1e9, inter_alpha=0.0, inter_beta=1e9)
    even = _trace(zpp, ib=10**9, eb=10**9)
    assert zpp.estimate_latency(even, free, stages=2).total_seconds == 0.75 * 2.0
    # the as-ran trace keeps its message count; the what-if chunking multiplies it
    assert zpp.pipelined_seconds(tr, links, 1) == one.total_seconds
    assert zpp.pipelined_seconds(tr, links, 8) > zpp.estimate_latency(tr, links, stages=8).total_seconds
    assert zpp.estimate_latency(_trace(zpp, compute=0.5), links).compute_seconds == 0.5
    for bad in (dict(intra_alpha=-1.0), dict(inter_beta=0.0)):
        with pytest.raises(zpp.ValidationError):
            zpp.LinkParams(**bad)
    with pytest.raises(zpp.ValidationError):
        zpp.estimate_latency(tr, links, stages=0)
    with pytest.raises(zpp.ValidationError):
        zpp.optimal_stages(tr, links, max_stages=0)
