import importlib

from ._bind import reference

reference()
globals().update({k: v for k, v in vars(importlib.import_module("xft_reference.calibration")).items()
                  if k.isupper()})
