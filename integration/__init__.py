"""Bindings of the B200 LP library into the reference `tvlp` package."""
