// Forwarding header: the reference file name for the B200 drop-in API.
#pragma once
#include "spike_b200.hpp"
