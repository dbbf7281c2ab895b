// Forwarding header: the reference file name for the B200 drop-in API
// (Spike2x2Factors, factor_2x2, solve_2x2, spikes_2x2, band_corner).
#pragma once
#include "spike_b200.hpp"
