"""Thread-backed stand-in for the `greenlet` module (test infrastructure only).

The reference's deterministic "coop" engine (reference pkg/src/ring3pc/
runtime.py:209-230) imports `greenlet`, which is not installed in this image.
This shim reproduces the subset that scheduler relies on -- getcurrent(),
greenlet(run), .switch(*args), .dead -- by running each greenlet on its own
daemon thread and passing a baton (one Event per greenlet) so exactly one
runs at a time.  It is only ever put on sys.path by tools that execute the
read-only reference to produce golden vectors; the product never imports it.
"""

from __future__ import annotations

import threading

_tls = threading.local()


class GreenletExit(BaseException):
    pass


class greenlet:  # noqa: N801 - mirrors the real module's class name
    def __init__(self, run=None, parent=None):
        self.run = run
        self.parent = parent if parent is not None else getcurrent()
        self.dead = False
        self._ev = threading.Event()
        self._thread = None
        self._inbox = ()
        self._exc = None

    # -- internals ---------------------------------------------------------
    def _main(self, args):
        _tls.current = self
        try:
            self.run(*args)
        except BaseException as e:  # noqa: BLE001 - re-raised in parent
            self._exc = e
        finally:
            self.dead = True
            parent = self.parent
            while parent is not None and parent.dead:
                parent = parent.parent
            parent._inbox = ()
            parent._exc_from_child = self._exc
            parent._ev.set()

    def _wait_turn(self):
        self._ev.wait()
        self._ev.clear()
        exc = getattr(self, "_exc_from_child", None)
        self._exc_from_child = None
        if exc is not None:
            raise exc
        return self._inbox

    # -- public API ----------------------------------------------------------
    def switch(self, *args):
        cur = getcurrent()
        if self.dead:
            return None
        if self._thread is None and self.run is not None and self is not cur:
            self._thread = threading.Thread(target=self._main, args=(args,),
                                            daemon=True)
            self._thread.start()
        else:
            self._inbox = args
            self._ev.set()
        got = cur._wait_turn()
        if len(got) == 0:
            return None
        return got[0] if len(got) == 1 else got


def getcurrent() -> greenlet:
    cur = getattr(_tls, "current", None)
    if cur is None:
        cur = greenlet.__new__(greenlet)
        cur.run = None
        cur.parent = None
        cur.dead = False
        cur._ev = threading.Event()
        cur._thread = threading.current_thread()
        cur._inbox = ()
        cur._exc = None
        _tls.current = cur
    return cur
