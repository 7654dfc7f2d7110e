import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# Debugging aid (DELTA_HANG_DEBUG=seconds): the attention backward writes
# per-CTA progress words to mapped host memory; a watchdog prints them and
# exits if one test runs longer than the given time (a hung kernel cannot be
# interrupted from Python).
_HANG = float(os.environ.get("DELTA_HANG_DEBUG", "0") or 0)
if _HANG > 0:
    import threading
    import time as _time

    _state = {"t0": None, "name": None, "buf": None}

    @pytest.fixture(autouse=True)
    def _hang_watch(request):
        if _state["buf"] is None:
            import ctypes

            import torch
            from paper_2203_15980_b200._lib import lib
            _state["buf"] = torch.zeros(4096 * 32, dtype=torch.int32).pin_memory()
            lib.delta_attention_debug.argtypes = [ctypes.c_void_p]
            lib.delta_attention_debug(_state["buf"].data_ptr())

            def _watch():
                while True:
                    _time.sleep(1)
                    t0 = _state["t0"]
                    if t0 and _time.time() - t0 > _HANG:
                        print(f"\nHANG in {_state['name']}; progress words:", flush=True)
                        for c, row in enumerate(_state["buf"].view(-1, 32).tolist()[:64]):
                            if any(row):
                                print(c, [hex(x) for x in row[:17]], flush=True)
                        os._exit(3)
            threading.Thread(target=_watch, daemon=True).start()
        _state["name"] = request.node.nodeid
        _state["t0"] = _time.time()
        yield
        _state["t0"] = None
