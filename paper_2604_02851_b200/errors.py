"""Exception types of the reference API (ref pkg/src/splatstream/protocol/framing.py:18)."""


class ProtocolError(Exception):
    pass
