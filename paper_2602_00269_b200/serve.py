"""Streaming wire + HTTP frontend + load-test client.

* ``ChunkFrame`` wire format: each frame is a 4-byte
  big-endian length, a fixed binary header -- request_id u64, chunk_index u32,
  available_at_ms u64 (server clock), playback_ms u32, flags u32 (bit 0 is_final,
  bit 1 error) -- and the payload: the chunk's REAL audio as 24 kHz mono 16-bit
  little-endian PCM (the reference specifies real-sized silence because its engine
  produces no audio).  SPEC.md:695 calls the header "24-byte" but lists five fields
  of 28 bytes; the field list is what is implemented.
* ``VoxServer``: ``POST /v1/generate`` (JSON {"prompt_tokens", "output_tokens"}) answers
  with a chunked stream of frames terminated by the is_final frame; ``GET /v1/metrics``
  (the reference MetricsReport of the served trace, core.py:300-333) and
  ``GET /v1/healthz``.  400 on a malformed body or 0 output tokens, 429 beyond the live
  request cap, 503 while draining.  One asyncio loop accepts
  connections; the StreamingEngine runs its own thread (engine.serve) and hands each
  request's chunks to that request's response writer by message passing
  (SPEC.md:725).
* ``load_test``: Poisson arrivals (the reference ``workload.build_workload``) against a
  server; client-observed frame times build a reference ``core.Trace`` so TTFA and
  viability come from the reference metric code.
"""

from __future__ import annotations

import asyncio
import json
import queue
import struct
import threading
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._ref import core

HEADER = struct.Struct(">QIQII")
LENGTH = struct.Struct(">I")
FLAG_FINAL = 1
FLAG_ERROR = 2
SAMPLE_RATE = 24000


@dataclass(frozen=True)
class ChunkFrame:
    request_id: int
    chunk_index: int
    available_at_ms: int
    playback_ms: int
    payload: bytes
    is_final: bool = False
    error: bool = False

    def encode(self) -> bytes:
        flags = (FLAG_FINAL if self.is_final else 0) | (FLAG_ERROR if self.error else 0)
        body = HEADER.pack(self.request_id, self.chunk_index, self.available_at_ms, self.playback_ms, flags)
        return LENGTH.pack(len(body) + len(self.payload)) + body + self.payload

    @staticmethod
    def decode_stream(buf: bytes) -> tuple[list["ChunkFrame"], bytes]:
        """Parse every complete frame at the front of buf; returns (frames, remainder)."""
        out = []
        off = 0
        while len(buf) - off >= LENGTH.size:
            (n,) = LENGTH.unpack_from(buf, off)
            if len(buf) - off - LENGTH.size < n:
                break
            rid, idx, at, pb, flags = HEADER.unpack_from(buf, off + LENGTH.size)
            p0 = off + LENGTH.size + HEADER.size
            out.append(ChunkFrame(rid, idx, at, pb, bytes(buf[p0:off + LENGTH.size + n]),
                                  bool(flags & FLAG_FINAL), bool(flags & FLAG_ERROR)))
            off += LENGTH.size + n
        return out, bytes(buf[off:])


def pcm16(x: np.ndarray) -> bytes:
    return np.clip(np.rint(np.asarray(x, np.float32) * 32767.0), -32768, 32767).astype("<i2").tobytes()


class VoxServer:
    """HTTP streaming service over one StreamingEngine (one GPU, one engine loop)."""

    def __init__(self, engine, host: str = "127.0.0.1", port: int = 0, max_live: Optional[int] = None):
        self.engine = engine
        self.host, self.port = host, port
        self.max_live = max_live or min(engine.policy.max_live_requests, engine.dev.cfg.max_slots)
        self.inbox: queue.Queue = queue.Queue()
        self.stop = threading.Event()
        self.draining = False
        self._streams: dict[int, asyncio.Queue] = {}
        self._arrival_ms: dict[int, float] = {}
        self._next_id = 0
        self._live = 0
        self._loop: Optional[asyncio.AbstractEventLoop] = None
        self._server = None
        self._thread: Optional[threading.Thread] = None
        self.engine_error: Optional[BaseException] = None
        engine.on_chunk = self._on_chunk

    # ------------------------------------------------------------------ engine side
    def _on_chunk(self, rid, index, avail_us, playback_us, pcm, final):
        frame = ChunkFrame(rid, index, int(avail_us // 1000), int(round(playback_us / 1000)),
                           pcm16(pcm) if pcm is not None else b"", final)
        q = self._streams.get(rid)
        if q is not None and self._loop is not None:
            self._loop.call_soon_threadsafe(q.put_nowait, frame)

    def _engine_main(self):
        try:
            self.engine.serve(self.inbox, self.stop)
        except BaseException as e:  # surface to the HTTP side; never hang clients
            self.engine_error = e
            if self._loop is not None:
                for rid, q in list(self._streams.items()):
                    self._loop.call_soon_threadsafe(q.put_nowait, ChunkFrame(rid, 0, 0, 0, b"", True, True))

    def now_ms(self) -> float:
        return (time.perf_counter() - self.engine._t0) * 1e3

    # ------------------------------------------------------------------ HTTP side
    async def start(self):
        self._loop = asyncio.get_running_loop()
        self._thread = threading.Thread(target=self._engine_main, daemon=True)
        self._thread.start()
        while self.engine._t0 == 0.0 and self.engine_error is None:
            await asyncio.sleep(0.001)
        self._server = await asyncio.start_server(self._handle, self.host, self.port)
        self.port = self._server.sockets[0].getsockname()[1]
        return self

    async def shutdown(self, drain_timeout_s: float = 30.0):
        """Graceful: refuse new requests (503), let live streams finish, stop the engine."""
        self.draining = True
        t0 = time.perf_counter()
        while self._live and time.perf_counter() - t0 < drain_timeout_s:
            await asyncio.sleep(0.01)
        self.stop.set()
        if self._thread is not None:
            await asyncio.get_running_loop().run_in_executor(None, self._thread.join, drain_timeout_s)
        if self._server is not None:
            self._server.close()
            await self._server.wait_closed()

    @staticmethod
    async def _reply(w, code: int, reason: str, body: bytes = b"", ctype: str = "application/json"):
        w.write(f"HTTP/1.1 {code} {reason}\r\nContent-Type: {ctype}\r\nContent-Length: {len(body)}\r\n"
                f"Connection: close\r\n\r\n".encode() + body)
        await w.drain()
        w.close()

    async def _handle(self, reader: asyncio.StreamReader, w: asyncio.StreamWriter):
        try:
            head = await reader.readuntil(b"\r\n\r\n")
        except (asyncio.IncompleteReadError, asyncio.LimitOverrunError):
            w.close()
            return
        lines = head.decode("latin-1").split("\r\n")
        try:
            method, path, _ = lines[0].split(" ", 2)
        except ValueError:
            await self._reply(w, 400, "Bad Request", b'{"error": "bad request line"}')
            return
        hdrs = {k.strip().lower(): v.strip() for k, v in (ln.split(":", 1) for ln in lines[1:] if ":" in ln)}
        body = await reader.readexactly(int(hdrs.get("content-length", "0") or 0))
        if method == "GET" and path == "/v1/healthz":
            await self._reply(w, 200, "OK", json.dumps({"ok": self.engine_error is None}).encode())
        elif method == "GET" and path == "/v1/metrics":
            tr = core.Trace(requests=list(self.engine.trace.requests), chunks=list(self.engine.trace.chunks))
            try:
                rep = core.build_report(tr).to_json().encode()
            except Exception as e:  # an empty trace has no report yet
                rep = json.dumps({"error": str(e)}).encode()
            await self._reply(w, 200, "OK", rep)
        elif method == "POST" and path == "/v1/generate":
            await self._generate(body, w)
        else:
            await self._reply(w, 404, "Not Found", b'{"error": "no such endpoint"}')

    async def _generate(self, body: bytes, w: asyncio.StreamWriter):
        try:
            req = json.loads(body or b"{}")
            P = int(req.get("prompt_tokens", 50))
            T = int(req["output_tokens"])
            if P < 1 or T < 1 or P + T + 1 > self.engine.dev.cfg.max_ctx:
                raise ValueError("prompt_tokens >= 1, output_tokens >= 1 and within the context capacity")
        except (ValueError, KeyError, TypeError, json.JSONDecodeError) as e:
            await self._reply(w, 400, "Bad Request", json.dumps({"error": str(e)}).encode())
            return
        if self.draining or self.engine_error is not None:
            await self._reply(w, 503, "Service Unavailable", b'{"error": "draining"}')
            return
        if self._live >= self.max_live:
            await self._reply(w, 429, "Too Many Requests", b'{"error": "max_live_requests exceeded"}')
            return
        rid = self._next_id
        self._next_id += 1
        q: asyncio.Queue = asyncio.Queue()
        self._streams[rid] = q
        self._live += 1
        arrival = self.now_ms()
        self.inbox.put((rid, P, T))
        w.write(("HTTP/1.1 200 OK\r\nContent-Type: application/octet-stream\r\nTransfer-Encoding: chunked\r\n"
                 f"X-Vox-Request-Id: {rid}\r\nX-Vox-Arrival-Ms: {arrival:.3f}\r\nConnection: close\r\n\r\n").encode())
        try:
            while True:
                f = await q.get()
                data = f.encode()
                w.write(f"{len(data):x}\r\n".encode() + data + b"\r\n")
                await w.drain()
                if f.is_final:
                    break
            w.write(b"0\r\n\r\n")
            await w.drain()
        except (ConnectionError, asyncio.CancelledError):
            pass
        finally:
            self._streams.pop(rid, None)
            self._live -= 1
            w.close()


# ---------------------------------------------------------------------- client
async def generate(host: str, port: int, output_tokens: int, prompt_tokens: int = 50, t0: float = 0.0):
    """One streaming request; returns (status, server arrival ms, [(client_ms, frame)])."""
    r, w = await asyncio.open_connection(host, port)
    body = json.dumps({"prompt_tokens": prompt_tokens, "output_tokens": output_tokens}).encode()
    w.write(f"POST /v1/generate HTTP/1.1\r\nHost: {host}\r\nContent-Type: application/json\r\n"
            f"Content-Length: {len(body)}\r\n\r\n".encode() + body)
    await w.drain()
    head = (await r.readuntil(b"\r\n\r\n")).decode("latin-1").split("\r\n")
    status = int(head[0].split(" ")[1])
    hdrs = {k.strip().lower(): v.strip() for k, v in (ln.split(":", 1) for ln in head[1:] if ":" in ln)}
    frames = []
    if status != 200:
        w.close()
        return status, None, frames
    buf = b""
    while True:
        size = int((await r.readuntil(b"\r\n")).strip(), 16)
        if size == 0:
            break
        buf += await r.readexactly(size)
        await r.readexactly(2)
        got, buf = ChunkFrame.decode_stream(buf)
        now = (time.perf_counter() - t0) * 1e3
        frames += [(now, f) for f in got]
        if any(f.is_final for f in got):
            break
    w.close()
    return status, float(hdrs.get("x-vox-arrival-ms", "nan")), frames


async def load_test(host: str, port: int, spec) -> dict:
    """Poisson arrivals of ``spec`` (reference workload.WorkloadSpec) against a server;
    client-observed frame times -> reference core metrics.  Connection failures are
    recorded per request and reported separately from the latency stats."""
    from ._ref import workload

    arrivals = workload.build_workload(spec)
    t0 = time.perf_counter()
    results = {}

    async def one(i, a):
        await asyncio.sleep(max(0.0, a.arrival_us / 1e6 - (time.perf_counter() - t0)))
        sent = (time.perf_counter() - t0) * 1e3
        try:
            results[i] = (sent, a) + await generate(host, port, a.target_output_tokens, a.prompt_tokens, t0)
        except (OSError, asyncio.IncompleteReadError) as e:
            results[i] = (sent, a, None, None, repr(e))

    await asyncio.gather(*(one(i, a) for i, a in enumerate(arrivals)))
    tr = core.Trace()
    errors, rejected, gaps, audio = {}, 0, [], {}
    for i, (sent, a, status, s_arr, frames) in sorted(results.items()):
        if status is None:
            errors[i] = frames
            continue
        if status != 200:
            rejected += 1
            continue
        req = core.Request(id=i, arrival_us=int(sent * 1000), prompt_tokens=a.prompt_tokens,
                           target_output_tokens=a.target_output_tokens)
        tr.requests.append(req)
        for t_ms, f in frames:
            tr.chunks.append(core.ChunkEvent(request=i, index=f.chunk_index, available_us=int(t_ms * 1000),
                                             playback_us=f.playback_ms * 1000, new_tokens=1))
        if frames:
            audio[frames[0][1].request_id] = np.frombuffer(b"".join(f.payload for _, f in frames), "<i2")
            req.first_chunk_us = int(frames[0][0] * 1000)
            req.phase = core.Phase.FINISHED if frames[-1][1].is_final and not frames[-1][1].error else \
                core.Phase.STEADY_STATE
            req.chunks_emitted = len(frames)
            # client TTFA - server TTFA = delivery overhead
            gaps.append((frames[0][0] - sent) - (frames[0][1].available_at_ms - s_arr))
    tr.chunks.sort(key=lambda c: (c.available_us, c.request, c.index))
    rep = core.build_report(tr) if tr.requests else None
    return {"report": rep.to_json_dict() if rep else None, "requests": len(arrivals), "errors": errors,
            "rejected": rejected, "client_minus_server_ttfa_ms": gaps, "trace": tr,
            "audio": audio}  # server request id -> the streamed int16 PCM
