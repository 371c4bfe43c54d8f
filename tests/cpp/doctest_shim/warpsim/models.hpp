// TEST INFRASTRUCTURE: maps the reference test files' #include "warpsim/models.hpp" onto the
// drop-in headers (include/warpsim_b200.hpp, include/warpsim_ir_b200.hpp).
#pragma once
#include "warpsim_b200.hpp"
#include "warpsim_ir_b200.hpp"
