"""HTTP sessions over the device engine (§8(f) row 4): the reference
service's contract (pkg/tests/test_service.py) -- health, 422 on bad
config, 404 on unknown sessions, 409 on busy sessions and failed steps,
state = the frame the engine writes -- through FastAPI's in-process client."""

import os

import pytest

fastapi = pytest.importorskip("fastapi")
from fastapi.testclient import TestClient  # noqa: E402

import paper_1805_08846_b200 as P  # noqa: E402
from paper_1805_08846_b200 import frames as F  # noqa: E402
from paper_1805_08846_b200.service import create_app  # noqa: E402

CFG = """[run]
problem = acoustics2d
t_end = 0.1
[grid]
cells = 40 32
[scheme]
limiter = mc
[boundary]
all = reflective
[initial]
profile = gaussian_pressure
width = 0.15
"""


@pytest.fixture
def client():
    return TestClient(create_app())


def test_health_and_errors_without_device(client):
    r = client.get("/healthz")
    assert r.status_code == 200 and r.json()["status"] == "ok"
    assert client.post("/sessions", json={"config_text": "[run]\nproblem = nope\n"}).status_code == 422
    assert client.post("/sessions", json={"config_text": ""}).status_code == 422
    assert client.get("/sessions/deadbeef").status_code == 404
    assert client.post("/sessions/deadbeef/evolve", json={"t_target": 1.0}).status_code == 404
    assert client.delete("/sessions/deadbeef").status_code == 404


@pytest.mark.gpu
def test_session_lifecycle_and_state_frames(client):
    r = client.post("/sessions", json={"config_text": CFG, "workers": 4, "tiles": "16x8"})
    assert r.status_code == 201, r.text
    info = r.json()
    sid = info["session_id"]
    assert info["cells"] == [40, 32] and info["num_states"] == 3 and info["time"] == 0.0
    r = client.post(f"/sessions/{sid}/evolve", json={"t_target": 0.05})
    assert r.status_code == 200
    ev = r.json()
    assert ev["time"] == 0.05 and ev["steps_accepted"] > 0
    state = client.get(f"/sessions/{sid}/state").content
    # the same run through the library
    with P.build_simulation(P.loads(CFG)) as sim:
        sim.run_until(0.05)
        assert state == F.frame_bytes(sim.grid, sim.t, sim.steps_accepted)
    fr = F.parse_frame(state)
    assert fr.time == 0.05 and fr.step == ev["steps_accepted"]
    assert client.post(f"/sessions/{sid}/evolve", json={"t_target": 0.01}).status_code == 422
    # busy: an operation while another holds the session lock
    sess = client.app.state.sessions.get(sid)
    sess.lock.acquire()
    try:
        assert client.post(f"/sessions/{sid}/evolve", json={"t_target": 0.06}).status_code == 409
        assert client.get(f"/sessions/{sid}/state").status_code == 409
    finally:
        sess.lock.release()
    assert client.delete(f"/sessions/{sid}").status_code == 204
    assert client.get(f"/sessions/{sid}").status_code == 404


@pytest.mark.gpu
def test_failed_step_is_409(client):
    sid = client.post("/sessions", json={"config_text": CFG}).json()["session_id"]
    sim = client.app.state.sessions.get(sid).sim
    sim.grid.interior(0)[3, 4] = float("nan")
    r = client.post(f"/sessions/{sid}/evolve", json={"t_target": 0.05})
    assert r.status_code == 409 and "non-finite" in r.json()["detail"]
    client.delete(f"/sessions/{sid}")


def test_device_fault_at_create_is_503_not_422(client, monkeypatch):
    # a CUDA failure while allocating the session is not invalid input
    from paper_1805_08846_b200 import service as S

    def boom(cfg, device=0):
        raise P.DeviceError("device allocation failed: out of memory")

    monkeypatch.setattr(S, "build_simulation", boom)
    r = client.post("/sessions", json={"config_text": CFG})
    assert r.status_code == 503 and "out of memory" in r.json()["detail"]
