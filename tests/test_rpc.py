"""The measurement pool's wire format (paper_1802_04799_b200/rpc.py) against
the reference's (R/src/rpc.cpp:62-82): length-prefixed JSON frames, a hello
greeting, id-echoing responses. The reference's own WorkerServer (run from
oracle/_ref) greets and answers our client's frames; our sm100 server serves
and our pool round-robins, retries and marks dead workers like the
reference's WorkerPool; on a GPU the server measures real Configs."""
import json
import os
import socket
import subprocess
import time

import pytest

from paper_1802_04799_b200 import _abi
from paper_1802_04799_b200.rpc import (WorkerPool, WorkerServer, desc_from_json, desc_to_json,
                                       recv_frame, send_frame)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "oracle", "_ref", "ref_driver")


def test_frame_round_trip_and_limit():
    a, b = socket.socketpair()
    with a, b:
        msg = {"id": "7", "config": {"tile_n": 64}, "text": "é" * 3}
        send_frame(a, msg)
        assert recv_frame(b) == msg
        # the header is the little-endian byte length of the JSON body
        send_frame(a, {"x": 1})
        hdr = b.recv(4)
        body = b.recv(64)
        assert int.from_bytes(hdr, "little") == len(body) and json.loads(body) == {"x": 1}
        b.sendall((70 << 20).to_bytes(4, "little"))
        with pytest.raises(_abi.TecError):
            recv_frame(a)


@pytest.mark.skipif(not os.path.exists(REF), reason="reference binary not built")
def test_reference_worker_speaks_our_framing():
    """The reference's WorkerServer greets our client and answers a request
    frame (an unparseable program -> its error response, id echoed)."""
    p = subprocess.Popen([REF, "serve", "20"], stdout=subprocess.PIPE, text=True)
    try:
        port = json.loads(p.stdout.readline())["port"]
        with socket.create_connection(("127.0.0.1", port), timeout=10) as s:
            hello = recv_frame(s)
            assert hello == {"hello": {"device": "vdla-sim", "version": 1}}
            send_frame(s, {"id": "42", "program": {"nope": True}, "target": "vdla", "repeats": 1})
            resp = recv_frame(s)
            assert resp["id"] == "42" and resp["status"] == "error" and resp["cost"] == 0.0
        pool = WorkerPool([f"127.0.0.1:{port}"], device_name="vdla-sim")
        r = pool.measure({"program": {}, "target": "vdla", "repeats": 1})
        assert r is not None and r["status"] == "error"
        pool.close()
    finally:
        p.kill()
        p.wait()


def test_sm100_server_and_pool_with_injected_measure():
    seen = []

    def fake(req):
        seen.append(req)
        if req["config"].get("tile_n") == 999:
            raise _abi.TecError(15, "no instance")
        return 10.0 + req["config"]["tile_n"]

    servers = [WorkerServer(measure=fake), WorkerServer(measure=fake)]
    try:
        pool = WorkerPool([f"127.0.0.1:{s.port}" for s in servers] + ["127.0.0.1:1"])
        d = _abi.ConvDesc(n=1, c=64, h=8, w=8, k=64, r=3, s=3, stride_h=1, stride_w=1, pad_h=1,
                          pad_w=1, depthwise=0, compute=_abi.COMPUTE_BF16)
        assert desc_from_json(desc_to_json(d)).k == 64
        costs = []
        for tn in (64, 128, 999, 999, 64):
            r = pool.measure({"target": "sm100", "desc": desc_to_json(d), "config": {"tile_n": tn},
                              "repeats": 2})
            if r is None:  # the dead third worker got this request
                continue
            costs.append((r["status"], r["cost"]))
        assert ("ok", 74.0) in costs and ("ok", 138.0) in costs and ("error", 0.0) in costs
        assert pool.alive() == 2  # the unreachable worker is marked dead
        pool.close()
    finally:
        for s in servers:
            s.stop()


@pytest.mark.gpu
def test_sm100_server_measures_configs_on_device():
    s = WorkerServer()
    try:
        pool = WorkerPool([f"127.0.0.1:{s.port}"])
        d = _abi.ConvDesc(n=8, c=64, h=28, w=28, k=64, r=3, s=3, stride_h=1, stride_w=1,
                          pad_h=1, pad_w=1, depthwise=0, compute=_abi.COMPUTE_BF16)
        r = pool.measure({"target": "sm100", "desc": desc_to_json(d), "config": {"tile_k": 1},
                          "repeats": 5})
        assert r["status"] == "ok" and r["cost"] > 0
        bad = pool.measure({"target": "sm100", "desc": desc_to_json(d),
                            "config": {"tile_m": 96}, "repeats": 1})
        assert bad["status"] == "error" and "LoweringError" in bad["detail"]
        pool.close()
    finally:
        s.stop()
