// decode.cpp — placeholder, replaced by the host decode loop.
#include "cascade.h"
extern "C" int cascade_decode(cascade_session*, const int32_t*, int, const cascade_decode_cfg*, int32_t*,
                              int32_t*, double*, int32_t, int32_t*) {
    return CASCADE_ERUNTIME;
}
