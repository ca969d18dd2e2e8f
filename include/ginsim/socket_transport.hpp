// ginsim/socket_transport.hpp -- the reference's header name for the socket
// bootstrap entry points (proj/core/include/ginsim/socket_transport.hpp:117-129):
// comm_init_socket and reserve_loopback_port live in runtime.hpp here (the
// GIN1-over-TCP transport itself is the Proxy backend's, csrc/net.cu).  This
// header lets reference sources that include it by name compile unchanged.
#pragma once

#include "ginsim/runtime.hpp"
