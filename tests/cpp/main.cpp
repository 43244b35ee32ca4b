// TEST INFRASTRUCTURE ONLY — entry point of the reference-unit-test runner.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
