// include/amqft/opmeter.hpp -- the reference's header name (proj/include/amqft/opmeter.hpp)
// resolved to the B200 library's declarations, so reference callers compile
// unchanged with -I<repo>/include ahead of their own include path.
#pragma once
#include "../amqft_b200.hpp"
