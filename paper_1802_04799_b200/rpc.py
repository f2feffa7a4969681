"""Cross-host measurement pool in the reference's RPC wire format
(R/src/rpc.cpp:62-82, R/include/tec/rpc.hpp:39-100).

Frames: a 4-byte little-endian length, then that many bytes of JSON (at most
64 MiB). A server greets every connection with {"hello": {"device": ...,
"version": 1}}, then answers one response frame per request frame, echoing
the request's "id" with "status" ("ok" | "error"), "cost" and "detail".

On a B200 the unit of measurement is a Config, not a LoopProgram: an sm100
worker (device "sm100") takes {"id", "target": "sm100", "desc": {conv
descriptor fields}, "epilogue": [op codes], "config": {knobs}, "repeats"} and
answers the tec_measure median in microseconds. Within one node the tuner
shards trials over local GPUs (tuner.measure) or ranks (parallel.py); this
pool reaches GPUs on other hosts with the same envelope as the reference's
vdla-sim workers, and the reference's own WorkerServer answers its framing
(tests/test_rpc.py).
"""
from __future__ import annotations

import json
import socket
import struct
import threading
from typing import Callable, Dict, List, Optional, Sequence

from . import _abi

MAX_FRAME = 64 << 20
VERSION = 1


def send_frame(sock: socket.socket, obj) -> None:
    body = json.dumps(obj, separators=(",", ":")).encode()
    if len(body) > MAX_FRAME:
        raise _abi.TecError(20, f"frame of {len(body)} bytes exceeds {MAX_FRAME}")
    sock.sendall(struct.pack("<I", len(body)) + body)


def _recv_all(sock: socket.socket, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            raise ConnectionError("peer closed the connection")
        buf += chunk
    return bytes(buf)


def recv_frame(sock: socket.socket):
    (n,) = struct.unpack("<I", _recv_all(sock, 4))
    if n > MAX_FRAME:
        raise _abi.TecError(20, f"frame of {n} bytes exceeds {MAX_FRAME}")
    return json.loads(_recv_all(sock, n).decode()) if n else None


def desc_to_json(d: _abi.ConvDesc) -> dict:
    return {f: int(getattr(d, f)) for f, _ in _abi.ConvDesc._fields_}


def desc_from_json(j: dict) -> _abi.ConvDesc:
    return _abi.ConvDesc(**{f: int(j[f]) for f, _ in _abi.ConvDesc._fields_})


def measure_request(req: dict, device: int = 0) -> float:
    """One sm100 measurement (tec_measure: L2-flushed launches, median us)."""
    import ctypes as C
    if req.get("target", "sm100") != "sm100":
        raise _abi.TecError(15, f"sm100 worker cannot measure target '{req.get('target')}'")
    d = desc_from_json(req["desc"])
    epi = _abi.Epilogue()
    ops = list(req.get("epilogue", [_abi.EPI_BIAS, _abi.EPI_RELU]))
    for i, op in enumerate(ops):
        epi.ops[i] = op
    epi.n_ops = len(ops)
    epi.bias = 1 if _abi.EPI_BIAS in ops else None
    epi.residual = 1 if _abi.EPI_ADD in ops else None
    kn = _abi.Knobs(**{k: int(v) for k, v in req.get("config", {}).items()})
    us = C.c_double(0)
    _abi.check(_abi.load().tec_measure(C.byref(d), C.byref(epi), C.byref(kn), device, 3,
                                       max(1, int(req.get("repeats", 10))), 1, C.byref(us)))
    return us.value


class WorkerServer:
    """Serves measurement requests on 127.0.0.1:port (0 = ephemeral), one
    connection at a time, like the reference's WorkerServer
    (R/src/rpc.cpp:129-181). `measure(req) -> cost` is injectable (tests)."""

    def __init__(self, port: int = 0, device: int = 0,
                 measure: Optional[Callable[[dict], float]] = None, name: str = "sm100"):
        self.name = name
        self.measure = measure or (lambda req: measure_request(req, device))
        self._ls = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        self._ls.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self._ls.bind(("127.0.0.1", port))
        self._ls.listen(8)
        self._ls.settimeout(0.2)
        self.port = self._ls.getsockname()[1]
        self._stop = threading.Event()
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def _run(self):
        while not self._stop.is_set():
            try:
                conn, _ = self._ls.accept()
            except (socket.timeout, OSError):
                continue
            with conn:
                conn.settimeout(10)
                try:
                    self._serve(conn)
                except (ConnectionError, OSError, ValueError):
                    pass

    def _serve(self, conn):
        send_frame(conn, {"hello": {"device": self.name, "version": VERSION}})
        while not self._stop.is_set():
            req = recv_frame(conn)
            resp = {"id": req.get("id", "") if isinstance(req, dict) else "", "cost": 0.0,
                    "detail": ""}
            try:
                resp["cost"] = float(self.measure(req))
                resp["status"] = "ok"
            except _abi.TecError as e:
                resp["status"], resp["detail"] = "error", str(e)
            except (KeyError, TypeError, ValueError) as e:
                resp["status"], resp["detail"] = "error", f"bad request: {e}"
            send_frame(conn, resp)

    def stop(self):
        self._stop.set()
        try:
            self._ls.close()
        except OSError:
            pass
        self._thr.join(timeout=2)


class WorkerPool:
    """Round-robin client over "host:port" workers (R/src/rpc.cpp:183-283):
    checks the greeting, retries once on a fresh connection, marks a worker
    dead after that; `measure` returns None when nobody is left (the caller
    then measures locally, as the reference does)."""

    def __init__(self, addrs: Sequence[str], device_name: str = "sm100"):
        self.device_name = device_name
        self.conns: List[Dict] = []
        for a in addrs:
            host, _, port = a.rpartition(":")
            if not host:
                raise _abi.TecError(20, f"worker address needs host:port, got {a}")
            self.conns.append({"host": host, "port": int(port), "sock": None, "dead": False})
        self._next = 0
        self._id = 0

    def alive(self) -> int:
        return sum(1 for c in self.conns if not c["dead"])

    def _connect(self, c) -> bool:
        if c["sock"] is not None:
            return True
        try:
            s = socket.create_connection((c["host"], c["port"]), timeout=10)
            hello = recv_frame(s)
            h = (hello or {}).get("hello", {})
            if h.get("device") != self.device_name or h.get("version") != VERSION:
                s.close()
                return False
            c["sock"] = s
            return True
        except (OSError, ConnectionError, ValueError):
            return False

    def measure(self, request: dict) -> Optional[dict]:
        live = [i for i in range(len(self.conns)) if not self.conns[(self._next + i) % len(self.conns)]["dead"]]
        if not live:
            return None
        c = self.conns[(self._next + live[0]) % len(self.conns)]
        self._next = (self._next + live[0] + 1) % len(self.conns)
        self._id += 1
        req = dict(request, id=str(self._id))
        for _ in range(2):
            if not self._connect(c):
                continue
            try:
                send_frame(c["sock"], req)
                resp = recv_frame(c["sock"])
                if isinstance(resp, dict) and resp.get("id") == req["id"]:
                    return resp
            except (OSError, ConnectionError, ValueError):
                pass
            c["sock"].close()
            c["sock"] = None
        c["dead"] = True
        return None

    def close(self):
        for c in self.conns:
            if c["sock"] is not None:
                c["sock"].close()
                c["sock"] = None
