"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtdb200.so")


def _load_gz_json(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def cases():
    return _load_gz_json("cases.json.gz")


@pytest.fixture(scope="session")
def vectors():
    return _load_gz_json("vectors.json.gz")


@pytest.fixture(scope="session")
def shardings():
    return _load_gz_json("shardings.json.gz")


@pytest.fixture(scope="session")
def layouts():
    return _load_gz_json("layouts.json.gz")


def trace_bytes(name: str) -> bytes:
    with gzip.open(os.path.join(GOLDEN, "traces", name + ".ttrc.gz"), "rb") as fh:
        return fh.read()


@pytest.fixture(scope="session")
def golden_trace_bytes():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = trace_bytes(name)
        return cache[name]
    return get


@pytest.fixture(scope="session")
def torchtap_golden():
    return _load_gz_json("torchtap.json.gz")
