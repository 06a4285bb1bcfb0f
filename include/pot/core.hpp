// Drop-in forwarding header: the reference API lives in pot/pot.hpp.
#pragma once
#include "pot.hpp"
