"""Remote worker serving the B200 detector over the reference's wire protocol
(reference ``tilepipe/distribution/worker.py`` and ``wire.py``).

A reference client (``evaluate_remote`` / ``run_remote_frame`` / ``run_stream``) talks
to ``DetectorServer`` unchanged; every EVAL_REQUEST's tiles go through the GPU detector
in ONE batched device call instead of one ``detect`` per crop.
"""

from .wire import ProtocolError, recv_message, send_message
from .worker import DetectorServer, serve

__all__ = ["DetectorServer", "ProtocolError", "recv_message", "send_message", "serve"]
