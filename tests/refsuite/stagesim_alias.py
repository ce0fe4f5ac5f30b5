"""pytest plugin: make ``import stagesim`` / ``import stagesim.<mod>`` resolve to
this package, so the reference's own test modules (/root/reference/pkg/tests)
run unmodified against the drop-in (`tests/test_reference_suite.py`)."""

from __future__ import annotations

import importlib
import importlib.abc
import importlib.util
import sys

TARGET = "paper_2504_08795_b200"


class _Alias(importlib.abc.MetaPathFinder, importlib.abc.Loader):
    _specs: dict = {}

    def find_spec(self, name, path=None, target=None):
        if name == "stagesim" or name.startswith("stagesim."):
            return importlib.util.spec_from_loader(name, self)
        return None

    def create_module(self, spec):
        real = importlib.import_module(TARGET + spec.name[len("stagesim"):])
        sys.modules[spec.name] = real
        self._specs[spec.name] = real.__spec__
        return real

    def exec_module(self, module):
        # the import machinery stamped the alias spec on the real module; put the
        # real one back so its own relative imports resolve against its package
        module.__spec__ = self._specs.pop(module.__spec__.name, module.__spec__)


sys.meta_path.insert(0, _Alias())
