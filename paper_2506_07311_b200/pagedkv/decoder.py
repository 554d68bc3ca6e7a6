"""pagedkv.decoder (reference decoder.py:196-287): the decode loop over the
paged cache.  Logits are numpy already (the model is numpy)."""

from ..decoder import DecodeSession, PagedDecoderCache  # noqa: F401
