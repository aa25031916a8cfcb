// include/amqft/variants.hpp -- the reference's header name (proj/include/amqft/variants.hpp)
// resolved to the B200 library's declarations, so reference callers compile
// unchanged with -I<repo>/include ahead of their own include path.
#pragma once
#include "../amqft_b200.hpp"
