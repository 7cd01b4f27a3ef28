"""Project store and HTTP service paths that never reach the GPU: parameter
parsing, data root, input validation and the error routes (the fills and
detection are covered by tests/ref_suite/test_ref_project.py and
test_ref_service.py on the GPU)."""

import math

import numpy as np
import pytest
from fastapi.testclient import TestClient

from paper_1611_05319_b200 import engine, project
from paper_1611_05319_b200.service import API, create_app


def _pgm(H, W):
    return f"P5\n{W} {H}\n255\n".encode() + bytes(H * W)


def _png(H, W):
    import io

    from PIL import Image

    buf = io.BytesIO()
    Image.fromarray(np.zeros((H, W, 3), dtype=np.uint8), mode="RGB").save(buf, format="PNG")
    return buf.getvalue()


def test_params_from_dict():
    p = engine.FillParams(r=4, mu=math.inf, order="onion", neighborhood="axis_ball",
                          g_source="fixed", g_fixed=(0.0, 1.0))
    assert project.params_from_dict(p.to_dict()) == p
    assert project.params_from_dict(None) == engine.FillParams()
    assert project.params_from_dict({"preset": "coherence_transport"}).g_source == \
        "modified_structure_tensor"
    for bad in ({"preset": "magic"}, {"radius": 3}, {"g_fixed": [1, 2, 3]}, {"order": "backwards"}):
        with pytest.raises(ValueError):
            project.params_from_dict(bad)


def test_store_validation_writes_nothing(tmp_path, monkeypatch):
    monkeypatch.setenv(project.DATA_DIR_ENV, str(tmp_path / "env"))
    assert project.data_root() == tmp_path / "env"
    with pytest.raises(project.DimensionMismatchError):
        project.create_project(_png(4, 5), _pgm(3, 2), tmp_path)
    with pytest.raises(ValueError):
        project.create_project(b"nope", _pgm(4, 5), tmp_path)
    with pytest.raises(ValueError):
        project.create_project(_png(4, 5), b"nope", tmp_path)
    assert project.list_projects(tmp_path) == []
    with pytest.raises(project.UnknownProjectError):
        project.open_project("missing", tmp_path)


def test_service_error_routes(tmp_path):
    with TestClient(create_app(tmp_path)) as c:
        assert c.get(API + "/projects").json() == {"projects": []}
        files = {"image": ("i.png", _png(4, 5), "image/png"),
                 "mask": ("m.pgm", _pgm(3, 2), "image/x-portable-graymap")}
        assert c.post(API + "/projects", files=files).status_code == 409
        files["image"] = ("i.png", b"nope", "image/png")
        assert c.post(API + "/projects", files=files).status_code == 400
        for url in ("splines", "result", "report", "guide-field", "image", "mask"):
            assert c.get(f"{API}/projects/nope/{url}").status_code == 404
        assert c.put(f"{API}/projects/nope/splines", content=b"{}").status_code == 404
        assert c.post(f"{API}/projects/nope/inpaint").status_code == 404
