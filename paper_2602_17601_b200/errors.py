"""Exception types shared with the reference API."""


class ConfigurationError(ValueError):
    """Bad shapes / configuration (mirrors ``gnnmpc.condensing.ConfigurationError``,
    ``condensing.py:36-37``)."""
