// fhp_b200/fhp.hpp — umbrella header of the C++ host layer (namespace
// fhp_b200), the B200 counterpart of the reference's proj/core/include/fhp.
#pragma once
#include "fhp_b200/bench.hpp"
#include "fhp_b200/checkpoint.hpp"
#include "fhp_b200/collision.hpp"
#include "fhp_b200/config.hpp"
#include "fhp_b200/engine.hpp"
#include "fhp_b200/lattice.hpp"
#include "fhp_b200/node_state.hpp"
#include "fhp_b200/observables.hpp"
#include "fhp_b200/step.hpp"
